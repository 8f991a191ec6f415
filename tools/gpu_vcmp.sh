#!/bin/bash
# outputs of variant libraries against the first one (max |delta| grey), config $CFG
mkdir -p gpurun_out
CFG=${CFG:-4}
for v in $VARS; do FABF_LIB=$PWD/vlibs/libfabf_$v.so timeout 300 python tools/dump_out.py $CFG /tmp/o_$v.npy; done
python - $VARS <<'PY' >> gpurun_out/vcmp_${TAG:-x}.log
import sys, numpy as np
v = sys.argv[1:]; a = np.load(f"/tmp/o_{v[0]}.npy")
for n in v[1:]:
    b = np.load(f"/tmp/o_{n}.npy"); print(n, "vs", v[0], "max|d|", float(np.max(np.abs(a.astype(np.float64) - b))), "n_diff", int(np.sum(a != b)))
PY
