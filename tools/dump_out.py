"""Write fabf_filter's output on one config (library in FABF_LIB) to an .npy
file, for comparing variant builds against each other: dump_out.py cfg path"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1811_02308_b200 as fb
import workloads

cfg, path = int(sys.argv[1]), sys.argv[2]
w = workloads.config(cfg)
plan = fb.Plan(*w.shape, int(os.environ.get("QFLAGS", "0")))
d = lambda a: torch.from_numpy(a).cuda()
out = fb.filter(plan, d(w.img), d(w.theta), d(w.sigma), w.rho, w.N)
torch.cuda.synchronize()
np.save(path, out.cpu().numpy())
