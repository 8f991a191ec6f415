#!/bin/bash
# config-5 cells (tools/time_c5.py) for variant libraries in VARS
mkdir -p gpurun_out
for v in $VARS; do
 for rep in 1 2; do
  name=${v%%:*}; envs=""; [ "$name" != "$v" ] && envs=${v#*:}; envs=${envs//,/ }
  env $envs FABF_LIB=$PWD/vlibs/libfabf_$name.so timeout 300 python tools/time_c5.py ${GEN:-texture} ${QN:-8} ${RHOS:-20 40} 2>&1 | sed "s/^/$v /" >> gpurun_out/c5_$TAG.log
 done
done
