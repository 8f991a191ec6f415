#!/bin/bash
# round evidence on one GPU: bench line, launch list of the bench command,
# ncu --set full of k_filter and k_bounds, config-5 sweep
mkdir -p gpurun_out
TAG=${TAG:-ev}
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch rc $?" >> gpurun_out/ncu_launch_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_kf_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_kf_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bounds -s 1 -c 1 -o gpurun_out/prof_kb_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_kb_$TAG.log 2>&1
if [ -z "$NOSWEEP" ]; then timeout 1200 python bench.py --sweep --steps 5 --warmup 3 > gpurun_out/sweep_$TAG.log 2>&1; fi
echo done >> gpurun_out/ncu_kb_$TAG.log
