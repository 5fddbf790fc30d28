"""Time operator applications (no per-kernel profiling events) for a config; prints ms/apply."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2306_17537_b200 as ie
from ie_workloads import make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--kernels", action="store_true", help="also print per-kernel ms (CUDA-event marks)")
a = ap.parse_args()
cfg = make_config(a.config)
ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, cfg.sigma_b, cfg.freq)
ie.ensure_workspace(ctx, nrhs=a.nrhs, restart=2)
ie.ie_set_contrast(ctx, torch.from_numpy(cfg.sigma()).cuda())
nx, ny, nz = cfg.n
x = torch.randn((a.nrhs, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    ie.ie_apply_operator(ctx, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(a.steps):
    ie.ie_apply_operator(ctx, x, y)
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{a.config} ms/apply {e0.elapsed_time(e1) / a.steps:.4f} "
      f"host-enqueue ms/apply {(t1 - t0) * 1e3 / a.steps:.4f} wall ms/apply {(t2 - t0) * 1e3 / a.steps:.4f}")
if a.kernels:
    ie.ie_profile(ctx, True)
    for _ in range(a.steps):
        ie.ie_apply_operator(ctx, x, y)
    torch.cuda.synchronize()
    prof = ie.ie_profile_read(ctx)
    ie.ie_profile(ctx, False)
    print(a.config, " ".join(f"{k.split()[0]} {v[0] / max(v[1], 1):.4f}" for k, v in prof.items() if v[1]))
