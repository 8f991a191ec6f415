#!/bin/bash
mkdir -p gpurun_out
for lib in paper_1811_02308_b200/libfabf.so variants/*.so; do
  FABF_LIB=$PWD/$lib timeout 300 python tools/time_cfg.py ${CFG:-4} >> gpurun_out/variants_${TAG:-x}.log 2>&1
done
