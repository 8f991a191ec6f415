#!/bin/bash
# time config CFG (default 4) for the default library and every variants/*.so
mkdir -p gpurun_out
for lib in paper_1811_02308_b200/libfabf.so variants/*.so; do
  echo "$lib $(FABF_LIB=$PWD/$lib timeout 300 python tools/time_cfg.py ${CFG:-4} 2>&1 | tail -1)" >> gpurun_out/vartime_${TAG:-x}.log
done
