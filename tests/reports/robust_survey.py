import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle, paper_1811_02308_b200 as fb, workloads
from parity import compare_guarded, grey_scale
oracle.build()
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
for kind in ("float", "voronoi", "texture"):
    for rho, N in ((2, 10), (5, 10), (10, 10), (20, 10), (40, 8), (20, 4)):
        w = workloads.random_case(1, 240, 320, seed=900 + rho + N, kind=kind, rho=rho, N=N)
        plan = fb.Plan(*w.shape)
        out = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
        torch.cuda.synchronize()
        o = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)
        mx, nbad, err = compare_guarded(out.cpu().numpy(), o, grey_scale(w.img))
        print(json.dumps({"kind": kind, "rho": rho, "N": N, "max": mx, "bad": nbad,
                          "fallback": plan.last_fallback_count()}), flush=True)
