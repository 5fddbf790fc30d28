"""Small driver for ncu: builds a config's context and applies the operator a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--gmres", type=int, default=0, help="also run this many full-domain GMRES iterations")
a = ap.parse_args()
cfg = make_config(a.config)
sigma = cfg.sigma()
ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
ie.ensure_workspace(ctx, nrhs=1, restart=cfg.restart)
ie.ie_set_contrast(ctx, torch.from_numpy(sigma).cuda())
ie.ie_set_source(ctx, np.array([cfg.sources[0][0]]), np.array([cfg.sources[0][1]]))
nx, ny, nz = cfg.n
x = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
ie.ie_get_incident(ctx, x)
y = torch.empty_like(x)
for _ in range(a.reps):
    ie.ie_apply_operator(ctx, x, y)
if a.gmres:
    e = torch.empty_like(x)
    st = ie.ie_solve_dd(ctx, e, "full", outer_tol=1e-30, restart=cfg.restart, max_iters=a.gmres, check=False)
    print(st["total_inner_iters"])
torch.cuda.synchronize()
print("ok")
