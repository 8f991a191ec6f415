"""Per-config report of the three oracles and the GPU path:

* O1 brute force eq.(1), O2 the __float128 reference (parity target), O3 the
  paper's Algorithm 1 as printed in fp64 (context): wall time on this host's
  cores (CPU model and thread count stated), on the whole image for configs
  1-4 and on 2 frames of a config-5 cell;
* how far O3 (the paper's own numerics) drifts from O2, in grey levels;
* PSNR against brute force: O2 literal / guarded, O3, and the CUDA path
  (literal / guarded / guarded + clamp) -- the paper's 40 dB bar;
* the paper's context: MATLAB 9.1 on a 3.4 GHz CPU, Table II.

GPU box:  python tests/reports/oracle_report.py > profiles/r2_oracle_report.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import oracle
import workloads

oracle.build()


def psnr(a, b, peak=255.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def timed(fn, *a, **k):
    t = time.perf_counter()
    r = fn(*a, **k)
    return r, time.perf_counter() - t


try:
    import torch

    gpu = torch.cuda.is_available()
    if gpu:
        import paper_1811_02308_b200 as fb
except Exception:
    gpu = False

print(json.dumps({"host": {"cpu_model": cpu_model(), "threads": os.cpu_count()},
                  "paper_context": "MATLAB 9.1, Linux, 3.4 GHz CPU, 32 GB (P:540); Table II (P:574-577), "
                                   "512x512 Gaussian omega: N=5 171-189 ms, brute force 3.90-12.4 s "
                                   "(22.8x at rho=3 .. 66.7x at rho=11); 'at least 20x' (P:90, P:564)"}),
      flush=True)
cases = [(workloads.config(c), str(c)) for c in (1, 2, 3, 4)]
w5 = workloads.config5(20, 8, batch=2, size=1024, generator="texture")
cases.append((w5, "5 (texture rho=20 N=8, 2 of 32 frames)"))
for w, cfg in cases:
    g1, t1 = timed(oracle.brute, w.img, w.theta, w.sigma, w.rho)
    o2, t2 = timed(oracle.fast, w.img, w.theta, w.sigma, w.rho, w.N)
    g3, t3 = timed(oracle.literal, w.img, w.theta, w.sigma, w.rho, w.N)
    drift = np.abs(g3 - o2["g_lit"])
    fin = np.isfinite(drift)
    px = int(w.img.size)
    rec = {"config": cfg, "case": w.name, "pixels": px, "rho": w.rho, "N": w.N,
           "seconds": {"O1_brute": round(t1, 2), "O2_fast_quad": round(t2, 2), "O3_literal_fp64": round(t3, 2)},
           "Mpix_s": {"O1_brute": px / t1 / 1e6, "O2_fast_quad": px / t2 / 1e6, "O3_literal_fp64": px / t3 / 1e6},
           "O3_vs_O2_literal_grey": {"max": float(np.max(drift[fin])) if fin.any() else None,
                                     "p99": float(np.quantile(drift[fin], 0.99)) if fin.any() else None,
                                     "nonfinite": int((~fin).sum())},
           "psnr_vs_brute": {"O2_literal": round(psnr(o2["g_lit"], g1), 2),
                             "O2_guarded": round(psnr(o2["g_guard"], g1), 2),
                             "O3_literal_fp64": round(psnr(np.where(fin, g3, 0), g1), 2)},
           "speedup_O1_over_O2": round(t1 / t2, 2), "speedup_O1_over_O3": round(t1 / t3, 2)}
    if gpu:
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
        for name, flags in (("literal", fb.FLAG_LITERAL), ("guarded", 0), ("guarded_clamp", fb.FLAG_CLAMP)):
            plan = fb.Plan(*w.shape, flags)
            out = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
            torch.cuda.synchronize()
            rec["psnr_vs_brute"]["gpu_" + name] = round(psnr(out.cpu().numpy(), g1), 2)
            plan.close()
    print(json.dumps(rec), flush=True)
