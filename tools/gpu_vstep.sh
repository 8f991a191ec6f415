#!/bin/bash
# whole-call timing (tools/time_step.py) of variant libraries, interleaved rounds
mkdir -p gpurun_out
TAG=${TAG:-vs}
for rep in 1 2 3; do
  for c in ${CFGS:-4}; do
    for v in $VARS; do
      name=${v%%:*}; envs=""; [ "$name" != "$v" ] && envs=${v#*:}; envs=${envs//,/ }
      env $envs FABF_LIB=$PWD/vlibs/libfabf_$name.so timeout 300 python tools/time_step.py $c 2>&1 | sed "s/^/$v /" >> gpurun_out/step_$TAG.log
    done
  done
done
