"""Probe block-Jacobi convergence on c5: e history for adaptive and fixed inner tolerances."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "c5")
ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
ie.ensure_workspace(ctx, boxes=cfg.boxes, nrhs=1, restart=cfg.restart)
ie.ie_set_contrast(ctx, torch.from_numpy(cfg.sigma()).cuda())
ie.ie_set_source(ctx, np.array([s for s, _ in cfg.sources]), np.array([m for _, m in cfg.sources]))
nx, ny, nz = cfg.n
e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
for scheme, adaptive, fixed in (("jacobi", True, 0), ("jacobi", False, 1e-8), ("gauss_seidel", True, 0)):
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-6, adaptive=adaptive, inner_tol_fixed=fixed,
                        restart=cfg.restart, max_sweeps=25, max_iters=3000, check=False)
    print(scheme, "adaptive" if adaptive else f"fixed {fixed}", st["sweeps"], ie.STATUS.get(st["status"]),
          " ".join(f"{v:.2e}" for v in st["e_hist"][:, 0]), flush=True)
