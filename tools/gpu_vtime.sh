#!/bin/bash
# time variant libraries (vlibs/libfabf_<name>.so) on config 4, interleaved
# rounds; optional quick parity on CHECK (a variant name); env per variant via
# "name:VAR=val"
mkdir -p gpurun_out
TAG=${TAG:-vt}
if [ -n "$CHECK" ]; then
  FABF_LIB=$PWD/vlibs/libfabf_$CHECK.so timeout 900 python tests/reports/quick_check.py > gpurun_out/quick_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/quick_$TAG.log
fi
for rep in 1 2 3; do
  for v in $VARS; do
    name=${v%%:*}; envs=""; [ "$name" != "$v" ] && envs=${v#*:}; envs=${envs//,/ }
    env $envs FABF_LIB=$PWD/vlibs/libfabf_$name.so timeout 300 python tools/time_cfg.py ${CFG:-4} 2>&1 | sed "s/^/$v /" >> gpurun_out/time_$TAG.log
  done
done
