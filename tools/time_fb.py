"""Time the exact-moment fallback stage on config-5 cases with many / few
flagged pixels (GPU box).  FABF_FB_MODE=0|1|2 selects auto / thread / warp."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1811_02308_b200 as fb
import workloads

cases = [("texture", 40, 10), ("texture", 40, 8), ("texture", 20, 8), ("texture", 20, 10),
         ("texture", 10, 10), ("texture", 5, 10), ("texture", 2, 10), ("rectangles", 40, 10),
         ("rectangles", 20, 10)]
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
for gen, rho, N in cases:
    w = workloads.config5(rho, N, batch=32, size=1024, generator=gen)
    plan = fb.Plan(*w.shape)
    img, th, sg = d(w.img), d(w.theta), d(w.sigma)
    out = torch.empty_like(img)
    for _ in range(2):
        fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
    st = np.zeros(4)
    for _ in range(5):
        _, ms = fb.filter_profile(plan, img, th, sg, w.rho, w.N, out=out)
        st += np.array(ms)
    st /= 5
    print(json.dumps({"mode": os.environ.get("FABF_FB_MODE", "0"), "gen": gen, "rho": rho, "N": N,
                      "fallback": int(plan.last_fallback_count()), "k_fallback_ms": round(st[3], 4),
                      "total_ms": round(float(st.sum()), 4)}), flush=True)
    plan.close()
