#!/bin/bash
# ncu capture of k_filter for a variant library (FABF_LIB)
mkdir -p gpurun_out
FABF_LIB=$PWD/$LIB python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/plain_$TAG.log 2>&1 && \
FABF_LIB=$PWD/$LIB ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc $?" >> gpurun_out/ncu_$TAG.log
