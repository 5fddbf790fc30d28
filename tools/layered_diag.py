"""Layered K-C' parity sweep: relative error of the GPU layered operator against the oracle on
random tables, for several grids and right-hand-side counts, under the kernel selected by
IE_ZLAYER_MODE (0 = TMA-ring DMMA for nz % 64 == 0, 1 = DMMA from global, 2 = DFMA)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

from oracle import physics, layered as lay
from test_gpu_layered import _cfg, _sigma, _ctx, _apply, _rand_field, rel

for n in [(4, 4, 64), (8, 8, 64), (2, 2, 64), (1, 1, 64), (2, 2, 128), (4, 4, 32)]:
    for nrhs in (1, 3):
        cfg = _cfg(n)
        rng = np.random.default_rng(2)
        Tq = lay.random_table(n, rng, scale=0.02)
        sig = _sigma(rng, n, cfg.sigma_b)
        ctx = _ctx(cfg, sig, table=Tq, nrhs=nrhs)
        x = _rand_field(rng, n, nrhs)
        y = _apply(ctx, x)
        A = lay.LayeredOperator(Tq, physics.contrast(sig, cfg.sigma_b))
        errs = [rel(y[r], A(x[r])) for r in range(nrhs)]
        # where is the error: per component and z
        r0 = y[0] - A(x[0])
        comp = [float(np.linalg.norm(r0[q]) / np.linalg.norm(y[0])) for q in range(3)]
        print(os.environ.get("IE_ZLAYER_MODE", "0"), n, nrhs, ["%.2e" % e for e in errs], ["%.1e" % c for c in comp], flush=True)
