"""Per-stage device time of config-5 cells (32 x 1024^2, sigma ~ U[5,60],
theta = f) for the library in FABF_LIB:  python tools/time_c5.py GEN N rho..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02308_b200 as fb, workloads
gen, N = sys.argv[1], int(sys.argv[2])
rhos = [int(r) for r in sys.argv[3:]] or [2, 5, 10, 20, 40]
w0 = workloads.config5(2, N, batch=32, size=1024, generator=gen)
d = lambda a: torch.from_numpy(a).cuda()
img, th, sg = d(w0.img), d(w0.theta), d(w0.sigma)
out = torch.empty_like(img)
plan = fb.Plan(*w0.shape, int(os.environ.get("QFLAGS", "0")))
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for rho in rhos:
    for _ in range(2):
        fb.filter(plan, img, th, sg, rho, N, out=out)
    st = np.zeros(4)
    K = 5
    for i in range(K):
        flush.fill_(float(i))
        _, ms = fb.filter_profile(plan, img, th, sg, rho, N, out=out)
        st += np.array(ms)
    st /= K
    print(json.dumps({"gen": gen, "N": N, "rho": rho, "stage_ms": [round(x, 4) for x in st.tolist()],
                      "total_ms": round(float(st.sum()), 4), "Gpix_s": w0.img.size / st.sum() / 1e6,
                      "fallback": plan.last_fallback_count()}), flush=True)
