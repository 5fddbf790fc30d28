"""Pins of oracle/gmres.py: dense LU truth, special cases, Born limit."""

import numpy as np
import pytest

from ie_workloads import make_config
from oracle import physics, operator as op
from oracle.gmres import gmres


def _setup(name):
    cfg = make_config(name)
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(cfg.sigma(), cfg.sigma_b)
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0 = np.stack([np.moveaxis(physics.incident_E(pts, s, m, k0, cfg.freq), -1, 0) for s, m in cfg.sources])
    return cfg, k0, ds, E0


class _Dense:
    def __init__(self, M):
        self.M = M

    def __call__(self, x):
        return (self.M @ x.ravel()).reshape(x.shape)


def test_gmres_identity_one_iteration():
    b = np.arange(12, dtype=complex).reshape(3, 2, 2, 1) + 1j
    x, info = gmres(lambda v: v, b, tol=1e-12)
    assert info["iters"] == 1 and info["converged"]
    assert np.abs(x - b).max() < 1e-14


def test_gmres_random_dense_system_vs_lu():
    rng = np.random.default_rng(4)
    n = 60
    M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    M = M / np.sqrt(n) * 0.5 + np.eye(n) * 2.0
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for restart in (5, 30, 80):
        x, info = gmres(_Dense(M), b, tol=1e-12, restart=restart)
        assert info["converged"]
        xs = np.linalg.solve(M, b)
        assert np.linalg.norm(x - xs) / np.linalg.norm(xs) < 1e-10
        assert info["relres_true"] <= 1e-12


def test_c1_gmres_matches_dense_lu():
    cfg, k0, ds, E0 = _setup("c1")
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    x_lu = np.linalg.solve(A, E0[0].ravel()).reshape(E0[0].shape)
    Op = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    x, info = gmres(Op, E0[0], x0=E0[0], tol=1e-10, restart=30)
    assert info["converged"] and info["relres_true"] <= 1e-10
    assert np.linalg.norm(x - x_lu) / np.linalg.norm(x_lu) < 1e-9
    # the discrete system is well conditioned (SURVEY 8c-6 reports cond ~ 5.9)
    assert np.linalg.cond(A) < 20


def test_zero_contrast_returns_incident_in_zero_iterations():
    cfg, k0, ds, E0 = _setup("c1")
    Op = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, np.zeros_like(ds))
    x, info = gmres(Op, E0[0], x0=E0[0], tol=1e-12)
    assert info["iters"] == 0 and info["converged"]
    assert np.array_equal(x, E0[0])


def test_born_limit_second_order():
    """E(eps dsigma) = E0 + eps G dsigma E0 + O(eps^2): the remainder falls 100x per decade."""
    cfg, k0, ds, E0 = _setup("c1")
    rem = []
    for eps in (1e-2, 1e-3):
        A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, eps * ds)
        E = np.linalg.solve(A, E0[0].ravel()).reshape(E0[0].shape)
        Op = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, eps * ds)
        born = E0[0] + Op.scatter(E0[0])
        rem.append(np.linalg.norm(E - born))
    ratio = rem[0] / rem[1]
    assert 80 < ratio < 125


def test_contraction_preconditioner_algebra_and_solution_invariance():
    """P a = I; isotropic sigma gives the scalar 2 sigma_b / (sigma + sigma_b); GMRES on
    (I - G dsigma) P chi = E0 returns E = P chi equal to the dense LU solution."""
    from oracle import preconditioner as pc
    cfg = make_config("c2mini")
    sigma = cfg.sigma()
    P = pc.contraction_P(sigma, cfg.sigma_b)
    a = (sigma + cfg.sigma_b * np.eye(3)) / (2 * cfg.sigma_b)
    assert np.abs(np.einsum("...ij,...jk->...ik", P, a) - np.eye(3)).max() < 1e-13
    s_iso = np.eye(3) * 0.7
    assert np.allclose(pc.contraction_P(s_iso, 0.1), 2 * 0.1 / (0.7 + 0.1) * np.eye(3), rtol=1e-15)
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(sigma, cfg.sigma_b)
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0 = np.moveaxis(physics.incident_E(pts, *cfg.sources[0], k0, cfg.freq), -1, 0)
    A = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    X = np.linalg.solve(op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds), E0.ravel()).reshape(E0.shape)

    class AP:
        def __call__(self, chi):
            return A(pc.apply_cellwise(P, chi))
    chi, info = gmres(AP(), E0, x0=pc.apply_cellwise(a, E0), tol=1e-12, restart=30)
    assert info["converged"]
    E = pc.apply_cellwise(P, chi)
    assert np.linalg.norm(E - X) < 1e-9 * np.linalg.norm(X)
    assert np.linalg.norm(E0 - A(E)) / np.linalg.norm(E0) < 1e-11  # the Eq. 9 residual


def test_gmres_converges_in_as_many_steps_as_distinct_eigenvalues():
    """Full GMRES on a normal matrix with d distinct eigenvalues reaches the exact solution in d
    Arnoldi steps (the minimal polynomial has degree d), and its least-squares residual estimate
    equals the true residual there -- pins the complex Givens rotations, not only the final answer."""
    rng = np.random.default_rng(5)
    lam = np.array([1.0 + 0.5j, 0.7 - 0.2j, 2.0 + 1.0j, 1.3 + 0.0j, 0.9 + 0.9j])
    n = 40
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    D = np.repeat(lam, n // len(lam))
    M = (Q * D) @ Q.conj().T
    b = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).reshape(n, 1, 1, 1)

    def A(v):
        return (M @ v.ravel()).reshape(v.shape)

    x, info = gmres(A, b, tol=1e-12, restart=30)
    assert info["converged"] and info["iters"] == len(lam)
    assert abs(info["relres_est"] - info["relres_true"]) < 1e-10
    # before the last step the estimate is the true least-squares residual of the Krylov space
    x4, info4 = gmres(A, b, tol=1e-30, restart=30, max_iters=4)
    assert abs(info4["relres_est"] - info4["relres_true"]) < 1e-10 * max(info4["relres_true"], 1e-300)


def test_background_conductivity_is_zero_contrast():
    """sigma = sigma_b I everywhere is no anomaly (dsigma = sigma - sigma_b I): the operator is
    the identity bitwise and the solve returns E0 in zero iterations."""
    n, h, sb, f = (4, 4, 4), (0.25, 0.25, 0.25), 0.7, 2e5
    k0 = physics.wavenumber(sb, f)
    sigma = np.broadcast_to(sb * np.eye(3), (4, 4, 4, 3, 3)).copy()
    ds = physics.contrast(sigma, sb)
    rng = np.random.default_rng(2)
    E = rng.standard_normal((3, 4, 4, 4)) + 1j * rng.standard_normal((3, 4, 4, 4))
    A = op.Operator(n, h, k0, sb, ds)
    assert np.array_equal(A(E), E)
    x, info = gmres(A, E, x0=E, tol=1e-12)  # warm start from E0 (Algorithm 1's initial iterate)
    assert info["iters"] == 0 and np.array_equal(x, E)
