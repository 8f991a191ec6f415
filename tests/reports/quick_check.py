"""Quick parity + timing on one degree (for FABF_ONLY_N development builds in
FABF_LIB): every pixel of small cases against the oracle, alpha/beta of the
diagnostic path bit-exact, then per-stage timing of config 4 (N=8)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1811_02308_b200 as fb
import workloads
from parity import compare_guarded

N = int(os.environ.get("QN", "8"))
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
cases = [workloads.config(4, scale=0.15), workloads.config(3, scale=0.3)]
for (kind, shape, rho) in [("voronoi", (2, 150, 140), 12), ("texture", (1, 131, 257), 5),
                           ("rect", (1, 200, 230), 96), ("texture", (1, 96, 200), 40),
                           ("rect", (1, 5, 300), 2), ("rect", (1, 7, 7), 3), ("rect", (1, 1, 1), 0),
                           ("float", (1, 57, 91), 3), ("flat", (1, 40, 40), 3), ("voronoi", (1, 577, 200), 40),
                           ("voronoi", (2, 300, 260), 20), ("texture", (1, 200, 333), 1), ("rect", (1, 66, 70), 4)]:
    cases.append(workloads.random_case(*shape, seed=7, kind=kind, rho=rho, N=N))
bad = 0
FLAGS = int(os.environ.get("QFLAGS", "0"))
for w in cases:
    plan = fb.Plan(*w.shape, FLAGS)
    out, dg = fb.filter_diag(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, N)
    out2 = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, N)
    torch.cuda.synchronize()
    o = oracle.fast(w.img, w.theta, w.sigma, w.rho, N)
    ra, rb = oracle.bounds(w.img, w.rho)
    sc = 1.0 if w.img.min() >= 0 and w.img.max() <= 255 and w.img.max() - w.img.min() > 64 else max(float(w.img.max() - w.img.min()), 1e-30) / 255
    mx, nbad, _ = compare_guarded(out.cpu().numpy(), o, sc)
    ab = np.array_equal(dg["alpha"].cpu().numpy(), ra) and np.array_equal(dg["beta"].cpu().numpy(), rb)
    same = torch.equal(out, out2)
    ok = nbad == 0 and ab and same
    bad += not ok
    print(json.dumps({"case": w.name, "shape": list(w.shape), "rho": w.rho, "max_grey": mx, "nbad": nbad,
                      "bounds_exact": ab, "diag_equals_plain": same, "fallback": plan.last_fallback_count(),
                      "ok": ok}), flush=True)
print("QUICK", "PASS" if bad == 0 else f"FAIL {bad}", flush=True)
