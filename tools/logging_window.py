"""The paper's moving-window logging simulation (section 3.3) on the B200:
one context for the window geometry (Green spectrum computed once, sigma0 = 0.1 S/m constant
per window), per station: window conductivity (host-generated, timed separately),
E0 of the axial transmitter, Algorithm 1 (GS-A, full-domain tolerance 1e-3 as in P:285) on 2
sub-domains along the hole, receivers at 7, 15, 30 m -> |H| along the tool axis (the paper's
|H_zz|)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import logging as lg


def run(n_stations=5, n=(256, 128, 128), h=0.25, scheme="gauss_seidel", tol=1e-3, precond=0, restart=50):
    origin, _ = lg.window_grid(n, h)
    nx, ny, nz = n
    boxes = [(0, nx // 2, 0, ny, 0, nz), (nx // 2, nx, 0, ny, 0, nz)]
    t0 = time.perf_counter()
    ctx = ie.ie_create(n, (h, h, h), origin, lg.SIGMA0, lg.FREQ)
    ie.ensure_workspace(ctx, boxes=boxes, nrhs=1, restart=restart)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    tx_w, m_w, rx_w = lg.tool_in_window()
    e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    rows = []
    for tx in lg.stations(n_stations):
        g0 = time.perf_counter()
        sig = torch.from_numpy(lg.window_sigma(tx, n, h)).cuda()
        torch.cuda.synchronize()
        gen = time.perf_counter() - g0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        ie.ie_set_contrast(ctx, sig)
        ie.ie_set_source(ctx, tx_w[None], m_w[None])
        st = ie.ie_solve_dd(ctx, e, scheme, boxes=boxes, outer_tol=tol, restart=restart, max_sweeps=30,
                            max_iters=1500, check=False, precond=precond)
        H, _ = ie.ie_receiver_fields(ctx, e, np.array(rx_w))
        ev1.record()
        torch.cuda.synchronize()
        rows.append(dict(tx=[round(v, 3) for v in tx], s=round(ev0.elapsed_time(ev1) / 1e3, 4), gen_s=round(gen, 3),
                         sweeps=st["sweeps"], iters=st["total_inner_iters"], e=st["e_final"],
                         status=ie.STATUS.get(st["status"]), Hax=[abs(H[0, r, 0]) for r in range(len(rx_w))]))
    return {"workload": f"moving window {nx}x{ny}x{nz} cells of {h} m, {scheme}{'+CIE' if precond else ''}, "
                        f"tol {tol}, {len(boxes)} sub-domains along the hole",
            "setup_s": round(setup, 3), "s_per_position": round(float(np.mean([r["s"] for r in rows])), 4),
            "generation_s_per_position": round(float(np.mean([r["gen_s"] for r in rows])), 3), "stations": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--stations", type=int, default=5)
    ap.add_argument("--scheme", default="gauss_seidel")
    ap.add_argument("--precond", type=int, default=0)
    ap.add_argument("--tol", type=float, default=1e-3)
    a = ap.parse_args()
    print(json.dumps(run(a.stations, scheme=a.scheme, precond=a.precond, tol=a.tol)))
