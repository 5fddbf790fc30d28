"""The CPU oracle's forward solves timed on the host cores (SURVEY 8(d) 'oracle timing beside
it'): the c5 full-domain solve (oracle GMRES(50) with the contraction-IE right preconditioner,
tol 1e-6 -- the bench's outer tolerance), a DD solve (Algorithm 1, GS-A, on c2mod, the oracle's
naive coupling schedule) and the c5 operator setup.  Writes profiles/r02_oracle_solves.json
(cited by bench.py's cpu_baseline).  Test infrastructure: runs the oracle only."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from ie_workloads import make_config
from oracle import physics, operator as op, gmres, preconditioner as pc, dd
from oracle._threads import WORKERS
import bench

out = {"cores": WORKERS, "cpu_model": bench.cpu_info()[1], "runs": []}
# c5 full-domain solve, contraction IE, tol 1e-6
cfg = make_config("c5")
sigma = cfg.sigma()
k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
ds = physics.contrast(sigma, cfg.sigma_b)
t0 = time.perf_counter()
A = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
t_setup = time.perf_counter() - t0
src, m = cfg.sources[0]
E0 = np.ascontiguousarray(np.moveaxis(physics.incident_E(physics.centroids(cfg.n, cfg.hvec, cfg.origin), src, m, k0,
                                                          cfg.freq), -1, 0))
P = pc.contraction_P(sigma, cfg.sigma_b)
t0 = time.perf_counter()
chi, info = gmres.gmres(lambda c: A(pc.apply_cellwise(P, c)), E0, tol=cfg.outer_tol, restart=cfg.restart, max_iters=400)
t_solve = time.perf_counter() - t0
out["runs"].append({"workload": "c5 full-domain GMRES(50) + contraction IE, tol 1e-6", "setup_s": round(t_setup, 1),
                    "solve_s": round(t_solve, 1), "iters": info["iters"], "relres_true": info["relres_true"],
                    "gpu_same_solve_s": "bench dd.full_gmres_cie (0.10 s)"})
print(json.dumps(out["runs"][-1]), flush=True)
del A, chi, P
# DD (GS-A) on c2mod
cfg = make_config("c2mod")
sigma = cfg.sigma()
k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
ds = physics.contrast(sigma, cfg.sigma_b)
E0 = np.ascontiguousarray(np.moveaxis(physics.incident_E(physics.centroids(cfg.n, cfg.hvec, cfg.origin),
                                                          cfg.sources[0][0], cfg.sources[0][1], k0, cfg.freq), -1, 0))
for scheme in ("gauss_seidel", "jacobi"):
    t0 = time.perf_counter()
    system = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, cfg.boxes)
    E, st = dd.solve_dd(system, E0, scheme, outer_tol=cfg.outer_tol, restart=cfg.restart)
    out["runs"].append({"workload": f"c2mod Algorithm 1 {scheme} (adaptive e/10), 2 z-boxes, tol {cfg.outer_tol}",
                        "solve_s": round(time.perf_counter() - t0, 2), "sweeps": st["sweeps"],
                        "inner_iters": st["total_inner_iters"], "converged": bool(st["converged"])})
    print(json.dumps(out["runs"][-1]), flush=True)
t0 = time.perf_counter()
x, info = gmres.gmres(op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds), E0, tol=cfg.outer_tol, restart=cfg.restart,
                      max_iters=3000)
out["runs"].append({"workload": f"c2mod full-domain GMRES({cfg.restart}), tol {cfg.outer_tol}",
                    "solve_s": round(time.perf_counter() - t0, 2), "iters": info["iters"]})
print(json.dumps(out["runs"][-1]), flush=True)
# the same c2mod solves on the GPU (one position: E0 + solve + receivers), for the same-config ratio
try:
    import torch
    import paper_2306_17537_b200 as ie
    if torch.cuda.is_available():
        ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
        ie.ensure_workspace(ctx, boxes=cfg.boxes, nrhs=1, restart=cfg.restart)
        ie.ie_set_contrast(ctx, torch.from_numpy(sigma).cuda())
        e = torch.empty((1, 3) + tuple(cfg.n[::-1]), dtype=torch.complex128, device="cuda")
        for scheme in ("full", "gauss_seidel", "jacobi"):
            ts = []
            for rep in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ie.ie_set_source(ctx, np.array([cfg.sources[0][0]]), np.array([cfg.sources[0][1]]))
                st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=cfg.outer_tol, restart=cfg.restart,
                                    max_sweeps=300, max_iters=3000, check=False)
                ie.ie_receiver_fields(ctx, e, np.array(cfg.receivers))
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            out["runs"].append({"workload": f"GPU c2mod {scheme}, tol {cfg.outer_tol} (E0 + solve + receivers)",
                                "solve_s": round(float(np.median(ts[1:])), 4), "iters": st["total_inner_iters"],
                                "sweeps": st["sweeps"], "status": ie.STATUS.get(st["status"])})
            print(json.dumps(out["runs"][-1]), flush=True)
except Exception as exc:  # no GPU here: the oracle timings stand alone
    out["gpu_error"] = repr(exc)
if "--c4" in sys.argv:
    # one c4mid station (31, 400 kHz, 3 RHS) with the physical table: oracle layered operator
    # (2-D FFT + dense z contraction) + GMRES(30) with the contraction IE, tol 1e-6
    from ie_workloads import layered_inputs as li
    from oracle import layered as lay
    cfg = make_config("c4mid")
    med = li.medium(cfg)
    t0 = time.perf_counter()
    T = li.table(cfg, med)
    t_table = time.perf_counter() - t0
    sig = cfg.sigma()
    sbz = lay.background_per_layer(cfg.n, cfg.origin, cfg.hvec, *cfg.background())
    dsl = lay.contrast_layered(sig, sbz)
    t0 = time.perf_counter()
    Al = lay.LayeredOperator(T, dsl)
    t_setup = time.perf_counter() - t0
    del T
    E0s = li.incident(cfg, med)
    Pl = pc.contraction_P(sig, np.broadcast_to(sbz[:, None, None], sig.shape[:3]))
    t0 = time.perf_counter()
    its = []
    for r in range(len(E0s)):
        chi, info = gmres.gmres(lambda c_: Al(pc.apply_cellwise(Pl, c_)), E0s[r], tol=cfg.outer_tol, restart=30,
                                max_iters=400)
        its.append(info["iters"])
    out["runs"].append({"workload": "c4mid station 31, 400 kHz, 3 RHS: oracle layered GMRES(30) + CIE, tol 1e-6",
                        "table_s": round(t_table, 1), "setup_s": round(t_setup, 1),
                        "solve_s": round(time.perf_counter() - t0, 1), "iters": its,
                        "gpu_same_solve_s": "c4 sweep c4mid@1e-06:full_gmres_cie per (station, frequency) unit"})
    print(json.dumps(out["runs"][-1]), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else
                    "profiles/r02_oracle_solves.json", "w"), indent=1)
