"""Accuracy survey of the CUDA path against the oracle on every pixel of a set
of cases (GPU box): max / p99.9 error in grey levels, counts above 0.01 and
0.025, and the worst pixels with their kappa, lambda, t0 and regime code.

  python tests/reports/err_survey.py [quick]
"""
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
from parity import compare_guarded, grey_scale

oracle.build()
quick = "quick" in sys.argv
cases = [workloads.config(1), workloads.config(2), workloads.config(3, scale=0.3),
         workloads.config(4, scale=0.2)]
if not quick:
    for gen in ("texture", "rectangles"):
        for rho, N in ((2, 10), (5, 10), (20, 10), (40, 4), (10, 6)):
            cases.append(workloads.config5(rho, N, batch=1, size=384, generator=gen))
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
for w in cases:
    plan = fb.Plan(*w.shape)
    out, dg = fb.filter_diag(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    dg = {k: v.cpu().numpy() for k, v in dg.items()}
    o = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    sc = grey_scale(w.img)
    mx, nbad, err = compare_guarded(out, o, sc)
    a, b = dg["alpha"].ravel().astype(np.float64), dg["beta"].ravel().astype(np.float64)
    lam = (b - a) ** 2 / (2 * w.sigma.ravel().astype(np.float64) ** 2)
    t0 = (w.theta.ravel() - a) / np.where(b > a, b - a, 1)
    worst = np.argsort(err)[-5:][::-1]
    rec = {"case": w.name, "px": int(err.size), "max": float(mx), "p999": float(np.quantile(err, 0.999)),
           "gt01": int((err > 0.01).sum()), "gt025": int((err > 0.025).sum()), "bad": nbad,
           "fallback": int(plan.last_fallback_count()),
           "worst": [{"err": float(err[i]), "kappa": float(o["kappa"].ravel()[i]),
                      "lam": float(lam[i]), "t0": float(t0[i]), "code": int(dg["code"].ravel()[i])}
                     for i in worst]}
    print(json.dumps(rec), flush=True)
