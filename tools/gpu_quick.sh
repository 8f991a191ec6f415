#!/bin/bash
# quick GPU iteration: optional pytest filter, then per-stage timing of one config
mkdir -p gpurun_out
TAG=${TAG:-q}
if [ -n "$PYTEST_K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
fi
for c in ${CFGS:-4}; do timeout 300 python tools/time_cfg.py $c >> gpurun_out/time_$TAG.log 2>&1; done
