#!/bin/bash
# ncu --set full capture of k_filter for a variant library, summarised on the box
# (details text, source CSV, op mix): LIB=vlibs/libfabf_x.so TAG=x [CFG=4]
mkdir -p gpurun_out
FABF_LIB=$PWD/$LIB python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/plain_$TAG.log 2>&1 && \
FABF_LIB=$PWD/$LIB ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc $?" >> gpurun_out/ncu_$TAG.log
R=gpurun_out/prof_$TAG.ncu-rep
ncu -i $R --page details > gpurun_out/details_$TAG.txt 2>&1
ncu -i $R --page source --csv --print-source cuda,sass 2> /dev/null | gzip -9 > gpurun_out/source_$TAG.csv.gz
python tools/ncu_ops.py $R > gpurun_out/ops_$TAG.txt 2>&1
rm -f $R
