#!/bin/bash
# iteration loop on the GPU box: tests (optionally filtered), bench, launch list
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --ref-pixels 2000 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
if [ -n "$PROF" ]; then
  python tools/run_cfg.py ${CFG:-4} 4 > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/run_cfg.py ${CFG:-4} 4 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_filter -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py ${CFG:-4} 4 > gpurun_out/ncu_$TAG.log 2>&1
  echo "prof rc $?" >> gpurun_out/ncu_$TAG.log
fi
