"""Run the filter a few times on one BASELINE config (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02308_b200 as fb
import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = workloads.config(cfg)
plan = fb.Plan(*w.shape, int(os.environ.get("QFLAGS", "0")))
d = lambda a: torch.from_numpy(a).cuda()
img, th, sg = d(w.img), d(w.theta), d(w.sigma)
out = torch.empty_like(img)
for _ in range(reps):
    fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
torch.cuda.synchronize()
print("ok", w.name, float(out.float().mean()))
