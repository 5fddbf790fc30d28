"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: the
operator on the c5 (256x256x128) and c4h (128x128x64) grids, sampled output cells checked
against the oracle's direct summation of Eq. 3 (one output cell at a time), plus
properties that hold at any size (linearity, zero contrast)."""

import numpy as np
import pytest

from ie_workloads import make_config
from oracle import physics, operator as op
from gpu_helpers import gpu_ctx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c5", "c4h"])
def test_fullsize_operator_sampled_cells(name):
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    sigma = cfg.sigma()
    ctx, _ = gpu_ctx(cfg, sigma=sigma, boxes=[], nrhs=1, restart=2)
    nx, ny, nz = cfg.n
    e0 = torch.empty((len(cfg.sources), 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    ie.ie_get_incident(ctx, e0)
    x = e0[:1].contiguous()
    y = torch.empty_like(x)
    ie.ie_apply_operator(ctx, x, y)
    torch.cuda.synchronize()
    xh = x.cpu().numpy()[0]
    yh = y.cpu().numpy()[0]
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(sigma, cfg.sigma_b)
    rng = np.random.default_rng(0)
    cells = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (nx // 2, ny // 2, nz // 2)]
    cells += [tuple(int(v) for v in rng.integers(0, [nx, ny, nz])) for _ in range(2)]
    ref = op.direct_rows(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, xh, cells)
    scale = np.abs(yh).max()
    for t, (cx, cy, cz) in enumerate(cells):
        got = yh[:, cz, cy, cx]
        assert np.abs(got - ref[t]).max() < 1e-11 * scale, (cells[t], got, ref[t])
    # linearity at full size: A(a x + b z) = a A x + b A z
    z = torch.roll(x, shifts=3, dims=4) * (0.5 - 0.25j)
    w = torch.empty_like(x)
    ie.ie_apply_operator(ctx, (2.0 + 1j) * x + z, w)
    v = torch.empty_like(x)
    ie.ie_apply_operator(ctx, z, v)
    lin = (2.0 + 1j) * y + v
    assert float(torch.linalg.vector_norm(w - lin) / torch.linalg.vector_norm(lin)) < 1e-13


@pytest.mark.parametrize("name,scheme", [("c5", "full"), ("c5", "gauss_seidel"), ("c4h", "full")])
def test_fullsize_solve_residual_at_sampled_cells(name, scheme):
    """Full-size forward solves as bench.py runs them: the Eq. 9 residual E0 - (I - G dsigma) E
    evaluated by the oracle's direct summation (one output cell at a time) at sampled cells is
    at the solver tolerance, and the library's reported e is <= outer_tol."""
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    sigma = cfg.sigma()
    ctx, _ = gpu_ctx(cfg, sigma=sigma, boxes=cfg.boxes, nrhs=len(cfg.sources), restart=cfg.restart)
    nx, ny, nz = cfg.n
    e = torch.empty((len(cfg.sources), 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    tol = 1e-7
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=tol, restart=cfg.restart, max_sweeps=100,
                        max_iters=3000)
    assert st["e_final"] <= tol
    e0 = torch.empty_like(e)
    ie.ie_get_incident(ctx, e0)
    E = e.cpu().numpy()[0]
    E0 = e0.cpu().numpy()[0]
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(sigma, cfg.sigma_b)
    rng = np.random.default_rng(1)
    cells = [(nx // 2, ny // 2, nz // 2)] + [tuple(int(v) for v in rng.integers(0, [nx, ny, nz])) for _ in range(2)]
    AE = op.direct_rows(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, E, cells)
    scale = np.linalg.norm(E0.ravel()) / np.sqrt(E0.size)  # rms of E0
    for t, (cx, cy, cz) in enumerate(cells):
        r = E0[:, cz, cy, cx] - AE[t]
        assert np.abs(r).max() < 100 * tol * max(scale, np.abs(E0[:, cz, cy, cx]).max()), (cells[t], r)


def test_slab_pipeline_matches_the_five_pass_schedule_bitwise():
    """The opt-in L2 slab pipeline (IE_SLABS=1) runs the same arithmetic per
    element on slab-local X2 buffers over three streams: identical output to the default path."""
    import os
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config("c4h")
    sigma = cfg.sigma()
    nx, ny, nz = cfg.n
    x = torch.randn((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    outs = []
    for slabs in ("0", "1"):
        os.environ["IE_SLABS"] = slabs
        try:
            ctx, _ = gpu_ctx(cfg, sigma=sigma, boxes=[], nrhs=1, restart=2)
        finally:
            os.environ.pop("IE_SLABS", None)
        y = torch.empty_like(x)
        ie.ie_apply_operator(ctx, x, y)
        torch.cuda.synchronize()
        outs.append(y.cpu())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("name", ["c5", "c4h"])
def test_fullsize_multi_rhs_equals_single_rhs(name):
    """Three right-hand sides in one application (the triaxial tool; the z-pass CTAs of one pencil
    tile for all RHS run together) give, per RHS, the single-RHS result bit for bit."""
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    ctx, _ = gpu_ctx(cfg, boxes=[], nrhs=3, restart=2)
    nx, ny, nz = cfg.n
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn((3, 3, nz, ny, nx), dtype=torch.complex128, device="cuda", generator=g)
    y3 = torch.empty_like(x)
    ie.ie_apply_operator(ctx, x, y3)
    for r in range(3):
        y1 = torch.empty_like(x[r:r + 1])
        ie.ie_apply_operator(ctx, x[r:r + 1].contiguous(), y1)
        assert torch.equal(y1[0], y3[r]), r


@pytest.mark.parametrize("name,boxes,precond", [("c5", False, 0), ("c4h", False, 1), ("c4h", True, 0),
                                                 ("c2mod", True, 1)])
def test_fused_passes_match_the_five_pass_schedule_bitwise(name, boxes, precond):
    """K-AB (K-A + K-B) and K-DE (K-D + K-E), each one persistent launch handing X1 through an
    L2-resident ring of plane buffers with per-slot producer/consumer counters, run the same
    per-element arithmetic as the separate passes: identical operator output for every on/off
    combination (IE_FUSED_AB / IE_FUSED_DE = 1 at context creation select the fused passes),
    on the grid and on every DD box (z-restricted sources included), with and without the
    contraction IE."""
    import os
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    sigma = cfg.sigma()
    outs = []
    for ab, de in (("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")):
        os.environ["IE_FUSED_AB"], os.environ["IE_FUSED_DE"] = ab, de
        try:
            ctx, _ = gpu_ctx(cfg, sigma=sigma, boxes=cfg.boxes if boxes else [], nrhs=1, restart=2)
        finally:
            os.environ.pop("IE_FUSED_AB", None)
            os.environ.pop("IE_FUSED_DE", None)
        res = []
        for b in (cfg.boxes if boxes else [None]):
            bn = (b[1] - b[0], b[3] - b[2], b[5] - b[4]) if b else cfg.n
            x = torch.randn((1, 3, bn[2], bn[1], bn[0]), dtype=torch.complex128, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(5))
            y = torch.empty_like(x)
            if precond:
                ie.ie_solve_subdomain(ctx, x, y.copy_(x), tol=1e-3, restart=2, max_iters=2, box=b, check=False,
                                      precond=1)
            else:
                ie.ie_apply_operator(ctx, x, y, box=b)
            torch.cuda.synchronize()
            res.append(y.cpu())
        outs.append(res)
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)
