"""Pins of oracle/dd.py (Algorithm 1, Eqs. 19-24, Appendix A)."""

import numpy as np
import pytest

from ie_workloads import make_config, box_grid
from oracle import physics, operator as op, dd
from oracle.gmres import gmres


def _setup(name):
    cfg = make_config(name)
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(cfg.sigma(), cfg.sigma_b)
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    s, m = cfg.sources[0]
    E0 = np.moveaxis(physics.incident_E(pts, s, m, k0, cfg.freq), -1, 0)
    return cfg, k0, ds, E0


def test_appendix_a_forward_substitution_equals_matrix_form():
    """Eq. A.5 (E^{k+1} = (D+L)^{-1}[E0 - U E^k]) equals Eqs. A.10-A.12 (sequential solves
    using the newest fields) on a 3-sub-domain dense instance."""
    cfg, k0, ds, E0 = _setup("c2mini")
    n = cfg.n
    boxes = [(0, 8, 0, 8, 0, 3), (0, 8, 0, 8, 3, 5), (0, 8, 0, 8, 5, 8)]
    A = op.dense_matrix(n, cfg.hvec, k0, cfg.sigma_b, ds)
    blocks, ids = dd.dense_blocks(A, n, boxes)
    rng = np.random.default_rng(0)
    Ek = E0.ravel() + 0.1 * (rng.standard_normal(E0.size) + 1j * rng.standard_normal(E0.size))
    seq = dd.dense_gs_sweep(blocks, [E0.ravel()[i] for i in ids], [Ek[i] for i in ids])
    mat = dd.dense_gs_matrix_form(A, ids, E0.ravel(), Ek)
    for b in range(3):
        assert np.linalg.norm(seq[b] - mat[ids[b]]) < 1e-12 * np.linalg.norm(mat)


def test_one_gs_sweep_equals_forward_substitution():
    """The oracle's matrix-free GS sweep (inner GMRES at tight tol, naive FFT couplings)
    reproduces the dense forward substitution of Appendix A."""
    cfg, k0, ds, E0 = _setup("c2mini")
    boxes = [(0, 8, 0, 8, 0, 3), (0, 8, 0, 8, 3, 5), (0, 8, 0, 8, 5, 8)]
    sysm = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, boxes)
    E1, st = dd.solve_dd(sysm, E0, "gauss_seidel", outer_tol=0.0, adaptive=False, inner_tol_fixed=1e-13,
                         max_sweeps=1)
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    blocks, ids = dd.dense_blocks(A, cfg.n, boxes)
    ref = dd.dense_gs_sweep(blocks, [E0.ravel()[i] for i in ids], [E0.ravel()[i] for i in ids])
    for b in range(3):
        assert np.linalg.norm(E1.ravel()[ids[b]] - ref[b]) < 1e-10 * np.linalg.norm(E0)


@pytest.mark.parametrize("name", ["c2mini", "c3mini", "c5mini"])
def test_jacobi_and_gs_converge_to_dense_solution(name):
    cfg, k0, ds, E0 = _setup(name)
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    x = np.linalg.solve(A, E0.ravel()).reshape(E0.shape)
    sysm = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, cfg.boxes)
    res = {}
    for scheme in ("jacobi", "gauss_seidel"):
        E, st = dd.solve_dd(sysm, E0, scheme, outer_tol=1e-10, restart=cfg.restart)
        assert st["converged"], (scheme, st["e_hist"])
        assert np.linalg.norm(E - x) / np.linalg.norm(x) < 1e-8
        res[scheme] = st
    # Table 1 ordering (soft): Jacobi needs at least as many sweeps as Gauss-Seidel
    assert res["jacobi"]["sweeps"] >= res["gauss_seidel"]["sweeps"]


def test_single_box_is_full_domain_gmres():
    cfg, k0, ds, E0 = _setup("c1")
    sysm = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds, [(0, 8, 0, 8, 0, 8)])
    E, st = dd.solve_dd(sysm, E0, "gauss_seidel", outer_tol=1e-10, restart=30)
    x, info = gmres(op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds), E0, x0=E0, tol=1e-11, restart=30)
    assert st["converged"]
    assert np.linalg.norm(E - x) / np.linalg.norm(x) < 1e-9


def test_zero_contrast_zero_sweeps():
    cfg, k0, ds, E0 = _setup("c2mini")
    sysm = dd.DDSystem(cfg.n, cfg.hvec, k0, cfg.sigma_b, np.zeros_like(ds), cfg.boxes)
    E, st = dd.solve_dd(sysm, E0, "jacobi", outer_tol=1e-12)
    assert st["sweeps"] == 0 and st["converged"]
    assert np.array_equal(E, E0)


def test_partition_validation():
    with pytest.raises(ValueError):
        dd.check_partition((4, 4, 4), [(0, 4, 0, 4, 0, 3), (0, 4, 0, 4, 2, 4)])
    dd.check_partition((4, 4, 4), box_grid((4, 4, 4), (2, 1, 2)))
