"""Layered-path (A3L) operator timing: the c3 grid (64^3) or c4 grid (128x128x64) with the
library's degenerate table (format 2), nrhs right-hand sides, per-kernel CUDA-event times."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3h")
ap.add_argument("--nrhs", type=int, default=3)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
cfg = make_config(a.config)
sigma = cfg.sigma()
ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq, table_format=2)
ie.ensure_workspace(ctx, nrhs=a.nrhs, restart=2)
ie.ie_set_contrast(ctx, torch.from_numpy(sigma).cuda())
nx, ny, nz = cfg.n
N = nx * ny * nz
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((a.nrhs, 3, nz, ny, nx)) + 0j).cuda()
y = torch.empty_like(x)
for _ in range(3):
    ie.ie_apply_operator(ctx, x, y)
torch.cuda.synchronize()
ie.ie_profile(ctx, True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    ie.ie_apply_operator(ctx, x, y)
e1.record()
torch.cuda.synchronize()
prof = ie.ie_profile_read(ctx)
ms = e0.elapsed_time(e1) / a.steps
R = 3 * nz
mbytes = (nx + 1) * (ny + 1) * R * R * 16
x2bytes = 2 * a.nrhs * 12 * N * 16
flops = 8 * R * R * 4 * nx * ny * a.nrhs  # complex MACs of the 4 NxNy columns x nrhs
kc = prof["K-C z-convolution"]
kc_ms = kc[0] / max(1, kc[1])
print(json.dumps({"config": a.config, "grid": cfg.n, "nrhs": a.nrhs, "ms_per_apply": ms,
                  "kernels_ms": {k: v[0] / max(1, v[1]) for k, v in prof.items()},
                  "kcprime": {"ms": kc_ms, "table_bytes": mbytes, "x2_bytes": x2bytes,
                              "gbs": (mbytes + x2bytes) / kc_ms / 1e6, "gflops": flops / kc_ms / 1e6}}))
