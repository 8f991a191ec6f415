#!/bin/bash
# accuracy survey + timing of the default library
mkdir -p gpurun_out
TAG=${TAG:-s}
timeout 900 python tests/reports/err_survey.py $QUICK > gpurun_out/survey_$TAG.log 2>&1
for c in ${CFGS:-4 3}; do timeout 300 python tools/time_cfg.py $c >> gpurun_out/survey_$TAG.log 2>&1; done
