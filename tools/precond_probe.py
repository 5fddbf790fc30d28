"""Iterations and time of full-domain GMRES / GS-A with and without the contraction-IE right
preconditioner on a config (default c5)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

for name in (sys.argv[1:] or ["c5"]):
    cfg = make_config(name)
    ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
    ie.ensure_workspace(ctx, boxes=cfg.boxes, nrhs=len(cfg.sources), restart=cfg.restart)
    ie.ie_set_contrast(ctx, torch.from_numpy(cfg.sigma()).cuda())
    ie.ie_set_source(ctx, np.array([s for s, _ in cfg.sources]), np.array([m for _, m in cfg.sources]))
    nx, ny, nz = cfg.n
    e = torch.empty((len(cfg.sources), 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    for scheme in ("full", "gauss_seidel", "jacobi", "fgmres_jacobi", "fgmres_gauss_seidel"):
        for pc in (0, 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=cfg.outer_tol, restart=cfg.restart,
                                max_sweeps=60, max_iters=3000, check=False, precond=pc, inner_tol_fixed=1e-2)
            torch.cuda.synchronize()
            print(name, scheme, "precond" if pc else "plain", st["total_inner_iters"], st["sweeps"],
                  f"{st['e_final']:.2e}", ie.STATUS.get(st["status"]), f"{time.perf_counter() - t0:.3f} s", flush=True)
