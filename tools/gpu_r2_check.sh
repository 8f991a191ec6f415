#!/bin/bash
# round-2 GPU check: the r1 library on the outlier-row regression (expected to
# fail), the whole -m gpu suite on the current library, then one bench line.
mkdir -p gpurun_out
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ -f vlibs/libfabf_r1.so ] && [ -z "$SKIP_OLD" ]; then
  FABF_LIB=vlibs/libfabf_r1.so timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k outlier \
    -p no:cacheprovider > gpurun_out/pytest_old_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/pytest_old_$TAG.log
fi
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS} -p no:cacheprovider -s > gpurun_out/pytest_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/bench_$TAG.log
