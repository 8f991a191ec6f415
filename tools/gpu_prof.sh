#!/bin/bash
# ncu evidence for one config: launch list + one full capture of k_filter
mkdir -p gpurun_out
CFG=${CFG:-4}
TAG=${TAG:-v1}
nvidia-smi -i 0 --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > gpurun_out/smi_test.csv 2> gpurun_out/smi_test.err &
SMI=$!
python tools/run_cfg.py $CFG 4 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/run_cfg.py $CFG 4 > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_filter -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/run_cfg.py $CFG 4 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc $?" >> gpurun_out/ncu_full_$TAG.log
kill $SMI
