#!/bin/bash
# development variant build: one degree (FABF_ONLY_N, default 8) -> vlibs/libfabf_$1.so
# (extra nvcc -D flags after the name); prints k_filter's registers / spills
mkdir -p vlibs
NAME=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -DFABF_ONLY_N=${QN:-8} -Xptxas -v "$@" -o vlibs/libfabf_$NAME.so paper_1811_02308_b200/csrc/fabf.cu 2> vlibs/build_$NAME.log
rc=$?
grep -A2 "Compiling entry function '_Z8k_filterILi${QN:-8}ELi11ELi128ELi2ELi0ELb0" vlibs/build_$NAME.log | grep -E "registers|spill" 
grep -E "error" vlibs/build_$NAME.log | head
exit $rc
