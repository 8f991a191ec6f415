import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1811_02308_b200 as fb, oracle, workloads
w = workloads.config(1)
plan = fb.Plan(*w.shape)
d = lambda a: torch.from_numpy(a).cuda()
out, dg = fb.filter_diag(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
torch.cuda.synchronize()
out = out.cpu().numpy(); dg = {k: v.cpu().numpy() for k, v in dg.items()}
o = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)
err = np.abs(out - o["g_guard"])
bad = np.argwhere(err[0] > 0.05)
print("nbad", len(bad))
ys, xs = bad[:, 0], bad[:, 1]
print("rows", np.unique(ys)[:50])
print("cols", np.unique(xs)[:50])
codes = dg["code"][0][err[0] > 0.05]
print("codes", np.unique(codes, return_counts=True))
print("good codes", np.unique(dg["code"][0][err[0] <= 0.05], return_counts=True))
for (y, x) in bad[:10]:
    print(y, x, out[0, y, x], o["g_guard"][0, y, x], dg["kappa"][0, y, x], o["kappa"][0, y, x], dg["code"][0, y, x])
