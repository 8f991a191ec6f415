#!/bin/bash
# accuracy survey + timing for every variants/*.so
mkdir -p gpurun_out
for lib in variants/*.so; do
  echo "== $lib" >> gpurun_out/varsurvey_${TAG:-x}.log
  FABF_LIB=$PWD/$lib timeout 600 python tests/reports/err_survey.py $QUICK >> gpurun_out/varsurvey_${TAG:-x}.log 2>&1
  for c in ${CFGS:-4 3}; do FABF_LIB=$PWD/$lib timeout 300 python tools/time_cfg.py $c >> gpurun_out/varsurvey_${TAG:-x}.log 2>&1; done
done
