import sys, time, json, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import paper_2306_17537_b200 as ie
from ie_workloads import logging as lg
n, h = (256, 128, 128), 0.25
origin, _ = lg.window_grid(n, h)
nx, ny, nz = n
ctx = ie.ie_create(n, (h, h, h), origin, lg.SIGMA0, lg.FREQ)
boxes = [(0, nx // 2, 0, ny, 0, nz), (nx // 2, nx, 0, ny, 0, nz)]
ie.ensure_workspace(ctx, boxes=boxes, nrhs=1, restart=50)
tx = lg.stations(3)[1]
sig = lg.window_sigma(tx, n, h)
print("sigma range", sig[..., 0, 0].min(), sig[..., 0, 0].max(), flush=True)
ie.ie_set_contrast(ctx, torch.from_numpy(sig).cuda())
txw, mw, rxw = lg.tool_in_window()
ie.ie_set_source(ctx, txw[None], mw[None])
e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
for pc in (0, 1):
    for restart in (30, 50):
        t = time.perf_counter()
        st = ie.ie_solve_dd(ctx, e, "full", outer_tol=1e-3, restart=restart, max_iters=2000, check=False, precond=pc)
        torch.cuda.synchronize()
        print("full", pc, restart, st["total_inner_iters"], st["e_final"], ie.STATUS.get(st["status"]), round(time.perf_counter() - t, 2), flush=True)
