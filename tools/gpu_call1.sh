#!/bin/bash
# round-2 evidence call: GPU suite, bench, ncu launch list + k_filter full capture
# (the .ncu-rep is summarised on the box and deleted: gpurun_out must stay < 64 MiB)
mkdir -p gpurun_out
TAG=${TAG:-base}
if [ -z "$NOTEST" ]; then
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
python tools/run_cfg.py 4 3 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py 4 3 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc $?" >> gpurun_out/ncu_$TAG.log
R=gpurun_out/prof_$TAG.ncu-rep
ncu -i $R --page details > gpurun_out/details_$TAG.txt 2>&1
python tools/ncu_ops.py $R > gpurun_out/ops_$TAG.txt 2>&1
python tools/ncu_lines.py $R 80 > gpurun_out/lines_$TAG.txt 2>&1
SORT=instr python tools/ncu_lines.py $R 80 > gpurun_out/lines_instr_$TAG.txt 2>&1
ncu -i $R --page source --csv --print-source cuda,sass > gpurun_out/source_$TAG.csv 2>&1
gzip -f gpurun_out/source_$TAG.csv
rm -f $R
ls -la gpurun_out
