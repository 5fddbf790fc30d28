"""GPU parity of the layered-background path (readings R17-R19): the packed
x-y spectra, the operator with K-C' (z-z' contraction per horizontal wavenumber) on
arbitrary and degenerate tables, the box operator, DD solves and the reciprocity receiver
form, each against oracle/layered.py."""

import numpy as np
import pytest

from ie_workloads import Config
from oracle import physics, layered as lay
from gpu_helpers import rel

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _cfg(n, h=0.2, sigma_b=0.5, freq=3e5):
    return Config("custom", n, h, sigma_b, freq, 0, None, sources=[])


def _sigma(rng, n, sb, s=0.3):
    nx, ny, nz = n
    A = rng.standard_normal((nz, ny, nx, 3, 3)) * s
    return 0.5 * (A + np.swapaxes(A, -1, -2)) + np.asarray(sb)[:, None, None, None, None] * np.eye(3) \
        if np.ndim(sb) else 0.5 * (A + np.swapaxes(A, -1, -2)) + sb * np.eye(3)


def _ctx(cfg, sigma, table=None, fmt=None, layers=None, z_iface=None, nrhs=1, boxes=None, restart=2):
    import torch
    import paper_2306_17537_b200 as ie
    ctx = ie.ie_create(cfg.n, cfg.hvec, cfg.origin, layers if layers is not None else cfg.sigma_b, cfg.freq,
                       table=table, table_format=fmt, z_iface=z_iface)
    ie.ensure_workspace(ctx, boxes=boxes, nrhs=nrhs, restart=restart)
    ie.ie_set_contrast(ctx, torch.from_numpy(np.ascontiguousarray(sigma)).cuda())
    return ctx


def _apply(ctx, x, box=None):
    import torch
    import paper_2306_17537_b200 as ie
    xd = torch.from_numpy(x).cuda()
    yd = torch.full_like(xd, np.nan)
    ie.ie_apply_operator(ctx, xd, yd, box=box)
    return yd.cpu().numpy()


def _rand_field(rng, n, nrhs):
    nx, ny, nz = n
    return rng.standard_normal((nrhs, 3, nz, ny, nx)) + 1j * rng.standard_normal((nrhs, 3, nz, ny, nx))


@pytest.mark.parametrize("n", [(8, 4, 4), (4, 8, 2), (2, 2, 8)])
def test_layer_spectrum_matches_oracle(n):
    import paper_2306_17537_b200 as ie
    cfg = _cfg(n)
    rng = np.random.default_rng(1)
    Tq = lay.random_table(n, rng)
    ctx = _ctx(cfg, _sigma(rng, n, cfg.sigma_b), table=Tq)
    got = ie.ie_get_layer_spectrum(ctx)
    nx, ny, nz = n
    M = lay.layered_spectra(Tq) / (4 * nx * ny)  # (3,3,nz,nz,2ny,2nx)
    ref = M[:, :, :, :, :ny + 1, :nx + 1].transpose(4, 5, 1, 3, 0, 2).reshape((ny + 1) * (nx + 1), 3 * nz, 3 * nz)
    assert rel(got, ref) < TOL


# nz = 64 / 128 run the TMA-ring DMMA kernel (k_zlayer_tma, 3nz/8 = 24 / 48 row tiles, the c3/c4
# path); nz = 32 and the deeper nz = 256 the DMMA-from-global kernel (the TMA ring is only
# instantiated for 64 and 128); the small shapes the DFMA kernel
@pytest.mark.parametrize("n", [(8, 4, 4), (4, 8, 2), (16, 8, 8), (8, 8, 32), (1, 2, 4), (4, 4, 64), (2, 2, 128),
                               (1, 2, 256)])
@pytest.mark.parametrize("nrhs", [1, 3, 5])
def test_layered_apply_matches_oracle_random_table(n, nrhs):
    cfg = _cfg(n)
    rng = np.random.default_rng(2)
    Tq = lay.random_table(n, rng, scale=0.02)
    sig = _sigma(rng, n, cfg.sigma_b)
    ctx = _ctx(cfg, sig, table=Tq, nrhs=nrhs)
    x = _rand_field(rng, n, nrhs)
    y = _apply(ctx, x)
    A = lay.LayeredOperator(Tq, physics.contrast(sig, cfg.sigma_b))
    for r in range(nrhs):
        assert rel(y[r], A(x[r])) < TOL


@pytest.mark.parametrize("n", [(16, 8, 8), (8, 8, 16), (16, 16, 64)])
def test_degenerate_tables_reproduce_the_homogeneous_operator(n):
    """format 2 (library-built degenerate table) and format 1 (the oracle's degenerate table)
    through K-C' equal the homogeneous K-A..K-E operator (Eq. 10)."""
    cfg = _cfg(n)
    rng = np.random.default_rng(3)
    sig = _sigma(rng, n, cfg.sigma_b)
    x = _rand_field(rng, n, 2)
    y_h = _apply(_ctx(cfg, sig, nrhs=2), x)
    y_2 = _apply(_ctx(cfg, sig, fmt=2, nrhs=2), x)
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    Tq = lay.homogeneous_table(n, cfg.hvec, k0, cfg.sigma_b)
    y_1 = _apply(_ctx(cfg, sig, table=Tq, nrhs=2), x)
    assert rel(y_2, y_h) < TOL and rel(y_1, y_h) < TOL


@pytest.mark.parametrize("n,box", [((16, 8, 8), (0, 8, 0, 4, 0, 4)), ((16, 8, 8), (8, 16, 4, 8, 4, 8)),
                                   ((16, 8, 8), (0, 16, 0, 8, 2, 4)),
                                   # 64-deep boxes of a 128-deep grid: the TMA-ring kernel with a
                                   # layer offset (the z-z' spectra depend on the box's first layer)
                                   ((4, 4, 128), (0, 4, 0, 4, 64, 128)), ((4, 4, 128), (0, 2, 2, 4, 0, 64))])
def test_layered_box_operator_is_the_diagonal_block(n, box):
    cfg = _cfg(n)
    rng = np.random.default_rng(4)
    Tq = lay.random_table(n, rng, scale=0.02)
    sig = _sigma(rng, n, cfg.sigma_b)
    ctx = _ctx(cfg, sig, table=Tq, boxes=[box])
    i0, i1, j0, j1, k0_, k1 = box
    bn = (i1 - i0, j1 - j0, k1 - k0_)
    x = _rand_field(rng, bn, 1)
    y = _apply(ctx, x, box=box)
    ds = physics.contrast(sig, cfg.sigma_b)[k0_:k1, j0:j1, i0:i1]
    A = lay.LayeredOperator(lay.box_table(Tq, box), ds)
    assert rel(y[0], A(x[0])) < TOL


def _layered_problem(n=(8, 8, 8)):
    """Two-layer background (sigma 0.6 below z = 0, 0.9 above) with a non-Toeplitz table:
    the degenerate table of 0.6 S/m plus a small seeded perturbation."""
    cfg = _cfg(n, h=0.25, sigma_b=0.6, freq=2e5)
    layers, z_if = [0.6, 0.9], [0.0]
    rng = np.random.default_rng(6)
    k0 = physics.wavenumber(0.6, cfg.freq)
    Tq = lay.homogeneous_table(n, cfg.hvec, k0, 0.6) + lay.random_table(n, rng, scale=1e-3)
    sbz = lay.background_per_layer(n, cfg.origin, cfg.hvec, layers, z_if)
    sig = np.abs(_sigma(rng, n, sbz, s=0.15))
    sig = 0.5 * (sig + np.swapaxes(sig, -1, -2))
    ds = lay.contrast_layered(sig, sbz)
    pts = physics.centroids(n, cfg.hvec, cfg.origin)
    src = [np.array([0.05, 0.03, 0.1]), np.array([0.0, -0.1, -0.2])]
    mom = [np.array([0.0, 0.0, 1.0]), np.array([1.0, 0.0, 0.0])]
    E0 = np.ascontiguousarray(np.stack([np.moveaxis(physics.incident_E(pts, s, m, k0, cfg.freq), -1, 0)
                                        for s, m in zip(src, mom)]))
    return cfg, layers, z_if, Tq, sig, ds, E0, k0, pts


@pytest.mark.parametrize("scheme", ["full", "jacobi", "gauss_seidel"])
def test_layered_solves_match_dense_lu(scheme):
    import torch
    import paper_2306_17537_b200 as ie
    cfg, layers, z_if, Tq, sig, ds, E0, k0, pts = _layered_problem()
    boxes = [(0, 8, 0, 8, 0, 4), (0, 8, 0, 8, 4, 8)] if scheme == "gauss_seidel" else \
        [(0, 4, 0, 8, 0, 4), (4, 8, 0, 8, 0, 4), (0, 4, 0, 8, 4, 8), (4, 8, 0, 8, 4, 8)]
    ctx = _ctx(cfg, sig, table=Tq, layers=layers, z_iface=z_if, nrhs=2, boxes=boxes, restart=30)
    with pytest.raises(ie.IEError):
        ie.ie_set_source(ctx, [[0.05, 0.03, 0.1]], [[0, 0, 1.0]])  # layered E0 is caller-supplied
    ie.ie_set_incident(ctx, torch.from_numpy(E0).cuda())
    A = lay.dense_matrix_layered(Tq, ds)
    X = np.stack([np.linalg.solve(A, e.ravel()).reshape(e.shape) for e in E0])
    e = torch.empty(E0.shape, dtype=torch.complex128, device="cuda")
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=boxes, outer_tol=1e-10, restart=30, max_sweeps=300)
    assert st["e_final"] <= 1e-10
    assert rel(e.cpu().numpy(), X) < 1e-6
    # receivers by reciprocity with the caller-supplied E0 of unit receiver dipoles
    rx = [np.array([0.1, 0.1, 0.6]), np.array([-0.2, 0.1, -0.6])]
    mr = [np.array([0.0, 0.0, 1.0]), np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 0.0])]
    dips = [(r, m) for r in rx for m in mr]
    e0rx = np.ascontiguousarray(np.stack([np.moveaxis(physics.incident_E(pts, r, m, k0, cfg.freq), -1, 0)
                                          for r, m in dips]))
    h0 = np.array([[m @ physics.incident_H(r, s, ms, k0) for (r, m) in dips]
                   for s, ms in zip([np.array([0.05, 0.03, 0.1]), np.array([0.0, -0.1, -0.2])],
                                    [np.array([0.0, 0.0, 1.0]), np.array([1.0, 0.0, 0.0])])])
    H = ie.ie_receiver_fields_table(ctx, e, torch.from_numpy(e0rx).cuda(), h0)
    dv = cfg.h ** 3
    for s in range(2):
        ref = np.array([lay.receiver_coupling(X[s], ds, e0rx[d], h0[s, d], dv, physics.omega_of(cfg.freq))
                        for d in range(len(dips))])
        assert rel(H[s], ref) < 1e-6


@pytest.mark.parametrize("scheme", ["full", "jacobi", "gauss_seidel"])
def test_deep_layered_solves_match_dense_lu(scheme):
    """A 128-deep two-layer grid split into two 64-deep boxes: every sub-domain apply runs the
    TMA-ring contraction with a layer offset (the upper box starts at layer 64)."""
    import torch
    import paper_2306_17537_b200 as ie
    n = (2, 2, 128)
    cfg, layers, z_if, Tq, sig, ds, E0, k0, pts = _layered_problem(n)
    boxes = [(0, 2, 0, 2, 0, 64), (0, 2, 0, 2, 64, 128)]
    ctx = _ctx(cfg, sig, table=Tq, layers=layers, z_iface=z_if, nrhs=2, boxes=boxes, restart=30)
    ie.ie_set_incident(ctx, torch.from_numpy(E0).cuda())
    A = lay.dense_matrix_layered(Tq, ds)
    X = np.stack([np.linalg.solve(A, e.ravel()).reshape(e.shape) for e in E0])
    e = torch.empty(E0.shape, dtype=torch.complex128, device="cuda")
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=boxes, outer_tol=1e-10, restart=30, max_sweeps=300)
    assert st["e_final"] <= 1e-10
    assert rel(e.cpu().numpy(), X) < 1e-6
