"""PSNR of the CUDA fast filter against brute force (eq.(1), the oracle's
fabfo_brute) per BASELINE config, three ways: literal eq.(29), guarded
(reading R7), guarded + clamp (north_star acceptance: "PSNR of the fast output
against brute force reported per config").  GPU box:

  python tests/reports/psnr_report.py > profiles/r1_psnr.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle
import paper_1811_02308_b200 as fb
import workloads

oracle.build()


def psnr(a, b, peak=255.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


cases = [(workloads.config(c), c) for c in (1, 2, 3, 4)]
for rho, N in ((2, 10), (10, 6), (20, 8)):
    cases.append((workloads.config5(rho, N, batch=1, size=1024), 5))
d = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
for w, cfg in cases:
    t = time.perf_counter()
    g = oracle.brute(w.img, w.theta, w.sigma, w.rho)
    tb = time.perf_counter() - t
    rec = {"config": cfg, "case": w.name, "pixels": int(w.img.size), "rho": w.rho, "N": w.N,
           "brute_seconds_cpu": round(tb, 1)}
    for name, flags in (("literal", fb.FLAG_LITERAL), ("guarded", 0), ("guarded_clamp", fb.FLAG_CLAMP)):
        plan = fb.Plan(*w.shape, flags)
        out = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
        torch.cuda.synchronize()
        rec["psnr_" + name] = round(psnr(out.cpu().numpy(), g), 2)
        plan.close()
    rec["psnr_input_vs_brute"] = round(psnr(w.img, g), 2)
    print(json.dumps(rec), flush=True)
