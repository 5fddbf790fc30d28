"""Per-iteration cost of the full-domain GMRES against the bare operator apply (host round trip
per Arnoldi step included): prints ms/iteration, ms/apply and the difference per config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

for name in sys.argv[1:] or ["c4h", "c5"]:
    cfg = make_config(name)
    ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
    ie.ensure_workspace(ctx, nrhs=1, restart=cfg.restart)
    ie.ie_set_contrast(ctx, torch.from_numpy(cfg.sigma()).cuda())
    ie.ie_set_source(ctx, np.array([s for s, _ in cfg.sources])[:1], np.array([m for _, m in cfg.sources])[:1])
    nx, ny, nz = cfg.n
    e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    x = torch.randn_like(e)
    y = torch.empty_like(e)
    for _ in range(3):
        ie.ie_apply_operator(ctx, x, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        ie.ie_apply_operator(ctx, x, y)
    torch.cuda.synchronize()
    t_apply = (time.perf_counter() - t0) / 20 * 1e3
    res = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = ie.ie_solve_dd(ctx, e, "full", outer_tol=1e-14, restart=cfg.restart, max_iters=40, check=False)
        torch.cuda.synchronize()
        res.append(((time.perf_counter() - t0) * 1e3, st["total_inner_iters"]))
    ms, it = res[-1]
    print(f"{name}: {it} iterations {ms:.1f} ms -> {ms / max(it, 1):.3f} ms/iteration; apply {t_apply:.3f} ms; "
          f"orthogonalisation + overhead {ms / max(it, 1) - t_apply:.3f} ms/iteration", flush=True)
