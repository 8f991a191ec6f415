"""Synthetic analogue of the paper's Table I and Fig.3:
PSNR (dB) of the fast filter against brute force eq.(1) for the classical
bilateral filter (theta = f, sigma = sigma_0 = 40) for N = 0..6 and rho in
{3, 5, 10}, beside Mozerov & van de Weijer's uniform-prior filter (the
comparison of Fig.3).  The paper's 512x512 photograph is not available:
a 512x512 config-3-style image (Voronoi + noise) and the texture generator
stand in; the paper's omega is a Gaussian on [-3 rho, 3 rho]^2, ours the box
of half-width rho (reading R1), so the rho columns are not the same windows.
The GPU path computes g-hat; the oracle computes brute force.  GPU box:

  python tests/reports/table1_analogue.py > profiles/r2_table1_analogue.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import oracle
import paper_1811_02308_b200 as fb
import workloads

PAPER = {3: [29.03, 35.16, 43.26, 50.28, 58.51, 67.58, 76.61], 5: [28.15, 32.87, 40.83, 47.56, 55.69, 64.99, 73.24],
         10: [27.49, 30.86, 38.21, 44.31, 52.19, 61.12, 68.04]}


def psnr(a, b, peak=255.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
images = {"voronoi512": workloads.voronoi(512, 512, seed=3512, n_seeds=64, noise_sd=15.0),
          "texture512": workloads.texture(512, 512, seed=2512)}
for name, f in images.items():
    f = np.asarray(f, np.float32).reshape(1, 512, 512)
    th = f.copy()
    sg = np.full_like(f, 40.0)
    for rho in (3, 5, 10):
        g = oracle.brute(f, th, sg, rho)
        plan = fb.Plan(*f.shape)
        row = {"image": name, "rho": rho, "sigma0": 40.0, "psnr_by_N": {}, "paper_table1_by_N": PAPER[rho]}
        for N in range(7):
            out = fb.filter(plan, d(f), d(th), d(sg), rho, N)
            torch.cuda.synchronize()
            row["psnr_by_N"][N] = round(psnr(out.cpu().numpy(), g), 2)
        moz = fb.filter_mozerov(plan, d(f), d(th), d(sg), rho)
        torch.cuda.synchronize()
        row["psnr_mozerov"] = round(psnr(moz.cpu().numpy(), g), 2)
        print(json.dumps(row), flush=True)
