"""Whole-call device time of fabf_filter on one config (no events inside the
call, L2 flushed between calls) for the library in FABF_LIB: median ms."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02308_b200 as fb
import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.config(cfg)
plan = fb.Plan(*w.shape, int(os.environ.get("QFLAGS", "0")))
d = lambda a: torch.from_numpy(a).cuda()
img, th, sg = d(w.img), d(w.theta), d(w.sigma)
out = torch.empty_like(img)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(5):
    fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
ts = []
for i in range(30):
    flush.fill_(float(i))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"lib": os.path.basename(os.environ.get("FABF_LIB", "default")), "cfg": cfg,
                  "ms_median": ts[len(ts) // 2], "ms_min": ts[0], "mpix_s": w.pixels / ts[len(ts) // 2] / 1e3}))
