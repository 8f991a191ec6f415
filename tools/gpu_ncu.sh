#!/bin/bash
# ncu --set full capture of one kernel (regex KREGEX) on config CFG
mkdir -p gpurun_out
TAG=${TAG:-n}
python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_filter} -s ${SKIP:-1} -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc $?" >> gpurun_out/ncu_$TAG.log
