#!/bin/bash
# ncu --set full of kernels matching KREGEX (each, -c 1) for the variant library
# VAR at config CFG; summaries on the box, reports deleted
mkdir -p gpurun_out
TAG=${TAG:-nv}
export FABF_LIB=$PWD/vlibs/libfabf_$VAR.so
python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/run_$TAG.log 2>&1
for k in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${k}_$TAG python tools/run_cfg.py ${CFG:-4} 3 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  R=gpurun_out/prof_${k}_$TAG.ncu-rep
  ncu -i $R --page details > gpurun_out/details_${k}_$TAG.txt 2>&1
  ncu -i $R --page source --csv --print-source cuda,sass 2> /dev/null | gzip -9 > gpurun_out/source_${k}_$TAG.csv.gz
  python tools/ncu_ops.py $R > gpurun_out/ops_${k}_$TAG.txt 2>&1
  rm -f $R
done
