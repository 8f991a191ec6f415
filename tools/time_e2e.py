"""e2e (fabf_filter_host, pinned host buffers) on config 4 for the band count
in FABF_HOST_BANDS: Mpix/s over 20 frames (GPU box)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02308_b200 as fb, workloads
w = workloads.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
plan = fb.Plan(*w.shape)
h = [torch.from_numpy(a).pin_memory() for a in (w.img, w.theta, w.sigma)]
ho = torch.empty_like(h[0]).pin_memory()
for _ in range(3):
    fb.filter_host(plan, *h, w.rho, w.N, ho)
t = time.perf_counter()
for _ in range(20):
    fb.filter_host(plan, *h, w.rho, w.N, ho)
dt = (time.perf_counter() - t) / 20
print(json.dumps({"bands": os.environ.get("FABF_HOST_BANDS", "8"), "ms": dt * 1e3, "mpix_s": w.pixels / dt / 1e6}))
