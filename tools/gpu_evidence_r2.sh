#!/bin/bash
# round-2 evidence (two calls: reports are ~20 MB each, gpurun_out <= 64 MiB)
#   PART=1: launch list of the bench command, ncu --set full of the default
#           k_filter and of k_bounds at config 4
#   PART=2: ncu --set full of the fused k_filter (FABF_FLAG_FUSED), config-5 sweep
mkdir -p gpurun_out
TAG=${TAG:-e1}
if [ "${PART:-1}" = 1 ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-other-configs"
  $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
  echo "launches rc $?" >> gpurun_out/plain_$TAG.log
  python tools/run_cfg.py 4 3 > gpurun_out/run4_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_kf_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_kf_$TAG.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_bounds -s 1 -c 1 -o gpurun_out/prof_kb_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_kb_$TAG.log 2>&1
  gzip -9 gpurun_out/*.ncu-rep
else
  QFLAGS=8 python tools/run_cfg.py 4 3 > gpurun_out/run4f_$TAG.log 2>&1 && \
  QFLAGS=8 ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_kff_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_kff_$TAG.log 2>&1
  gzip -9 gpurun_out/*.ncu-rep
  timeout 1500 python bench.py --sweep --steps 5 --warmup 2 > gpurun_out/sweep_$TAG.jsonl 2>&1
  echo "sweep rc $?" >> gpurun_out/sweep_$TAG.jsonl
fi
