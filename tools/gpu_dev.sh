#!/bin/bash
# development loop: quick parity of the library in FABF_LIB (one degree), then
# per-stage timing of config 4 for every library given in LIBS
mkdir -p gpurun_out
TAG=${TAG:-dev}
FABF_LIB=${CHECK_LIB:-$PWD/vlibs/libfabf_dev.so} timeout 900 python tests/reports/quick_check.py > gpurun_out/quick_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/quick_$TAG.log
for lib in ${LIBS:-vlibs/libfabf_dev.so}; do
  for c in ${CFGS:-4}; do
    FABF_LIB=$PWD/$lib timeout 300 python tools/time_cfg.py $c >> gpurun_out/time_$TAG.log 2>&1
  done
done
