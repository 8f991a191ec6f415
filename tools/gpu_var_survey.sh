#!/bin/bash
mkdir -p gpurun_out
for lib in paper_1811_02308_b200/libfabf.so variants/lamb8.so variants/lamb16.so; do
  echo "== $lib" >> gpurun_out/survey_L.log
  FABF_LIB=$PWD/$lib timeout 600 python tools/err_survey.py >> gpurun_out/survey_L.log 2>&1
  FABF_LIB=$PWD/$lib timeout 300 python tools/time_cfg.py 4 >> gpurun_out/survey_L.log 2>&1
done
