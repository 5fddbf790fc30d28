"""Literal c4 (400 kHz) at tol 1e-6: full-domain GMRES + contraction IE with restart 30 / 128
at a few stations (how far the 200x resistive slab of R23 is from convergence)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2306_17537_b200 as ie
from ie_workloads import make_config, layered_inputs as li
from ie_workloads.configs import c4_stations

cfg = make_config("c4")
med = li.medium(cfg)
T = li.table(cfg, med)
sig = torch.from_numpy(cfg.sigma()).cuda()
st_all = c4_stations()
for restart in (30, 128):
    ctx = bench._layered_ctx(cfg, T, sig, 3, [], restart)
    for s in (0, 31, 63):
        srcs = [(st_all[s]["tx"], m) for m in st_all[s]["moments"]]
        E0 = torch.from_numpy(li.incident(cfg, med, srcs)).cuda()
        ie.ie_set_incident(ctx, E0)
        e = torch.empty_like(E0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ie.ie_solve_dd(ctx, e, "full", outer_tol=1e-6, restart=restart, max_iters=6000, check=False, precond=1)
        torch.cuda.synchronize()
        print(json.dumps({"restart": restart, "station": s, "s": round(time.perf_counter() - t0, 3),
                          "iters": r["total_inner_iters"], "e_final": r["e_final"],
                          "status": ie.STATUS.get(r["status"])}), flush=True)
    del ctx
    torch.cuda.empty_cache()
