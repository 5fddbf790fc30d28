import sys, os, json, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2306_17537_b200 as ie
from ie_workloads import make_config
for name in ["c5", "c2mod"]:
    cfg = make_config(name)
    ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
    ie.ensure_workspace(ctx, nrhs=1, restart=cfg.restart)
    ie.ie_set_contrast(ctx, torch.from_numpy(cfg.sigma()).cuda())
    ie.ie_set_source(ctx, np.array([s for s, _ in cfg.sources]), np.array([m for _, m in cfg.sources]))
    nx, ny, nz = cfg.n
    e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    for tol in (1e-6, 1e-9):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = ie.ie_solve_dd(ctx, e, "full", outer_tol=tol, restart=cfg.restart, max_iters=3000, check=False)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(name, os.environ.get("IE_DGKS_ETA2", "0.5"), tol, st["total_inner_iters"], st["e_final"], round(t1 - t0, 3), flush=True)
