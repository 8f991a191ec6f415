#!/bin/bash
# round-2 evidence, second session: GPU suite, bench, launch list of the bench
# command, ncu --set full of k_filter and k_bounds at config 4.  The reports
# are summarised ON the box (details text, source CSV, traffic.json entries)
# and deleted: gpurun_out must stay under 64 MiB.
mkdir -p gpurun_out
TAG=${TAG:-f1}
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-other-configs"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
echo "launches rc $?" >> gpurun_out/plain_$TAG.log
python tools/run_cfg.py 4 3 > gpurun_out/run4_$TAG.log 2>&1
for k in k_filter k_bounds; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${k}_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  R=gpurun_out/prof_${k}_$TAG.ncu-rep
  ncu -i $R --page details > gpurun_out/details_${k}_$TAG.txt 2>&1
  ncu -i $R --page source --csv --print-source cuda,sass 2> /dev/null | gzip -9 > gpurun_out/source_${k}_$TAG.csv.gz
  python tools/ncu_ops.py $R > gpurun_out/ops_${k}_$TAG.txt 2>&1
done
if [ -n "$SWEEP" ]; then
  timeout 1500 python bench.py --sweep --steps 5 --warmup 2 > gpurun_out/sweep_$TAG.jsonl 2>&1
  echo "sweep rc $?" >> gpurun_out/sweep_$TAG.jsonl
fi
cp profiles/traffic.json gpurun_out/traffic_before_$TAG.json
python tools/ncu_traffic.py k_filter=gpurun_out/prof_k_filter_$TAG.ncu-rep k_bounds=gpurun_out/prof_k_bounds_$TAG.ncu-rep > gpurun_out/traffic_$TAG.log 2>&1
cp profiles/traffic.json gpurun_out/traffic_$TAG.json
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
