"""Block Jacobi on the c5 recipe, GPU vs oracle sweep by sweep: the e history
(Eq. 9 after every sweep) of the GPU's Algorithm 1 and of the oracle's (oracle/dd.py, naive
coupling schedule, scipy.fft on all host cores) on the same inputs, adaptive inner tolerance
e/10 and a fixed one, same stop rule (R16: e grows 3 sweeps in a row).  Writes JSON."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config
from oracle import physics, dd

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5jac")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--out", default="gpurun_out/jacobi_oracle_vs_gpu.json")
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--splits", default=None, help="box splits sx,sy,sz (default: the config's boxes)")
ap.add_argument("--n", default=None, help="grid nx,ny,nz overriding the config's (same recipe)")
a = ap.parse_args()
cfg = make_config(a.config)
if a.n:
    cfg.n = tuple(int(v) for v in a.n.split(","))
    out_n = cfg.n
if a.splits:
    from ie_workloads import box_grid
    cfg.boxes = box_grid(cfg.n, tuple(int(v) for v in a.splits.split(",")))
sigma = cfg.sigma()
out = {"config": a.config, "grid": list(cfg.n), "boxes": [list(b) for b in cfg.boxes], "outer_tol": cfg.outer_tol, "runs": []}
ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
ie.ensure_workspace(ctx, boxes=cfg.boxes, nrhs=1, restart=cfg.restart)
ie.ie_set_contrast(ctx, torch.from_numpy(sigma).cuda())
pos = np.array([s for s, _ in cfg.sources])
mom = np.array([m for _, m in cfg.sources])
ie.ie_set_source(ctx, pos, mom)
nx, ny, nz = cfg.n
e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
modes = (("adaptive", True, 0.0), ("fixed 1e-8", False, 1e-8))
for label, adaptive, fixed in modes:
    t0 = time.perf_counter()
    st = ie.ie_solve_dd(ctx, e, "jacobi", boxes=cfg.boxes, outer_tol=cfg.outer_tol, adaptive=adaptive,
                        inner_tol_fixed=fixed, restart=cfg.restart, max_sweeps=a.sweeps, max_iters=3000, check=False)
    out["runs"].append({"side": "gpu", "inner": label, "sweeps": st["sweeps"], "status": ie.STATUS.get(st["status"]),
                        "e_hist": [float(v) for v in st["e_hist"][:, 0]], "s": round(time.perf_counter() - t0, 2)})
    print(json.dumps(out["runs"][-1]), flush=True)
if not a.no_oracle:
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(sigma, cfg.sigma_b)
    E0 = np.ascontiguousarray(np.moveaxis(physics.incident_E(physics.centroids(cfg.n, cfg.hvec, cfg.origin),
                                                             pos[0], mom[0], k0, cfg.freq), -1, 0))
    system = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, cfg.boxes)
    for label, adaptive, fixed in modes[:1]:
        t0 = time.perf_counter()
        E, st = dd.solve_dd(system, E0, "jacobi", outer_tol=cfg.outer_tol, adaptive=adaptive, inner_tol_fixed=fixed,
                            restart=cfg.restart, max_sweeps=a.sweeps)
        out["runs"].append({"side": "oracle", "inner": label, "sweeps": st["sweeps"],
                            "status": "converged" if st["converged"] else "not converged",
                            "e_hist": [float(v) for v in st["e_hist"]], "s": round(time.perf_counter() - t0, 2)})
        print(json.dumps(out["runs"][-1]), flush=True)
json.dump(out, open(a.out, "w"))
