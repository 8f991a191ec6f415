import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_02308_b200 as fb
rho = int(sys.argv[1]); H = int(sys.argv[2]); W = int(sys.argv[3])
f = torch.from_numpy(np.random.default_rng(0).normal(100, 50, (1, H, W)).astype(np.float32)).cuda()
plan = fb.Plan(1, H, W)
try:
    a, b = fb.bounds(plan, f, rho)
    torch.cuda.synchronize()
    print("ok", rho, H, W)
except Exception as e:
    print("FAIL", rho, H, W, str(e)[:80])
