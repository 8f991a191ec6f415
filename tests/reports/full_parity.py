"""Every pixel of a full-size BASELINE config against the oracle (GPU box;
minutes of CPU for the oracle):  python tests/reports/full_parity.py 4 > profiles/r1_full_parity_cfg4.json

Reports max |delta| (grey), the count above 0.01 / 0.05, the bit-exactness of
alpha / beta (fabf_bounds vs the oracle's window scan) and the identity pixels."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1811_02308_b200 as fb
import workloads
from parity import compare_guarded

oracle.build()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.config(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
plan = fb.Plan(*w.shape)
out = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
a, b = fb.bounds(plan, d(w.img), w.rho)
torch.cuda.synchronize()
out = out.cpu().numpy()
t = time.perf_counter()
o = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)
to = time.perf_counter() - t
ra, rb = oracle.bounds(w.img, w.rho)
mx, nbad, err = compare_guarded(out, o, 1.0)
ident = (o["code"] & 1) > 0
print(json.dumps({
    "config": cfg, "case": w.name, "pixels": int(out.size), "max_abs_delta_grey": mx,
    "p999_grey": float(np.quantile(err, 0.999)), "pixels_above_0.01": int((err > 0.01).sum()),
    "pixels_above_0.05": nbad, "alpha_bit_exact": bool(np.array_equal(a.cpu().numpy(), ra)),
    "beta_bit_exact": bool(np.array_equal(b.cpu().numpy(), rb)),
    "identity_pixels": int(ident.sum()),
    "identity_exact": bool(np.array_equal(out.ravel()[ident.ravel()], w.img.ravel()[ident.ravel()])),
    "fallback_pixels": int(plan.last_fallback_count()), "oracle_seconds": round(to, 1),
    "oracle_threads": os.cpu_count()}))
