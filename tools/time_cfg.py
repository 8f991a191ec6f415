"""Time fabf_filter_profile on one config (default 4) for the library in FABF_LIB."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02308_b200 as fb, workloads
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.config(cfg)
plan = fb.Plan(*w.shape, int(os.environ.get("QFLAGS", "0")))
d = lambda a: torch.from_numpy(a).cuda()
img, th, sg = d(w.img), d(w.theta), d(w.sigma)
out = torch.empty_like(img)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
st = np.zeros(4)
K = 10
for i in range(K):
    flush.fill_(float(i))
    _, ms = fb.filter_profile(plan, img, th, sg, w.rho, w.N, out=out)
    st += np.array(ms)
st /= K
print(json.dumps({"lib": os.environ.get("FABF_LIB", "default"), "flags": os.environ.get("QFLAGS", "0"), "cfg": cfg, "stage_ms": st.tolist(),
                  "total_ms": float(st.sum()), "mpix_s": w.pixels / st.sum() / 1e3}))
L = fb.lib()
if hasattr(L, "fabf_exp_timers"):
    import ctypes
    arr = (ctypes.c_ulonglong * 8)()
    L.fabf_exp_timers(arr)  # reset
    fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
    L.fabf_exp_timers(arr)
    ctas = arr[6]
    names = ["centre", "prologue", "A", "B", "C1", "C2"]
    print(json.dumps({"lib": os.environ.get("FABF_LIB", "default"), "ctas": ctas,
                      "kcycles_per_cta": {n: arr[i] / max(1, ctas) / 1e3 for i, n in enumerate(names)}}))
