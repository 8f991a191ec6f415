#!/bin/bash
# texture-application tests on the default library, then whole-call timing of
# the variant libraries in $VARS (tools/gpu_vstep.sh)
mkdir -p gpurun_out
TAG=${TAG:-t1}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${PYTEST_K:-texture}" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
[ -n "$VARS" ] && bash tools/gpu_vstep.sh
true
