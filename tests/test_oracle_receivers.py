"""Pins of oracle/receivers.py (Eq. 4 with Eq. 6): reciprocity of the discrete system,
the reciprocity (E0-of-receiver) form, and the zero-contrast case."""

import numpy as np

from ie_workloads import make_config
from oracle import physics, operator as op, receivers


def _solve(cfg, k0, ds, src, m):
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0 = np.moveaxis(physics.incident_E(pts, src, m, k0, cfg.freq), -1, 0)
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    return np.linalg.solve(A, E0.ravel()).reshape(E0.shape)


def test_source_receiver_reciprocity():
    """m_r . H(r_r; m_s at r_s) = m_s . H(r_s; m_r at r_r) (Lorentz reciprocity of the
    discrete IE: K symmetric, dsigma symmetric)."""
    cfg = make_config("c1")
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(cfg.sigma(), cfg.sigma_b)
    # make it anisotropic so the check is not trivially diagonal
    ds[2:6, 2:6, 2:6, 0, 2] = ds[2:6, 2:6, 2:6, 2, 0] = 0.4
    rs, ms = np.array([0.0, 0.0, 1.0]), np.array([0.3, 0.0, 1.0])
    rr, mr = np.array([0.5, 0.25, -1.5]), np.array([1.0, -0.5, 0.2])
    Es = _solve(cfg, k0, ds, rs, ms)
    Er = _solve(cfg, k0, ds, rr, mr)
    Hr = receivers.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, Es, [rr], rs, ms)[0]
    Hs = receivers.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, Er, [rs], rr, mr)[0]
    a, b = mr @ Hr, ms @ Hs
    assert abs(a - b) < 1e-12 * abs(a)


def test_direct_form_equals_reciprocity_form():
    """m_r . H_scat(r) = (i omega mu0)^-1 sum_c E0_{m_r at r}(r_c) . J_c dv."""
    cfg = make_config("c2mini")
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(cfg.sigma(), cfg.sigma_b)
    src, m = cfg.sources[0]
    E = _solve(cfg, k0, ds, src, m)
    rx = np.array([0.05, 0.05, 0.95])
    mr = np.array([0.2, 1.0, -0.3])
    H = receivers.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, E, [rx], src, m)[0]
    Hs = H - physics.incident_H(rx, src, m, k0)
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0r = physics.incident_E(pts, rx, mr, k0, cfg.freq)  # (nz,ny,nx,3)
    J = np.moveaxis(op.contrast_source(ds, E), 0, -1)
    dv = cfg.h ** 3
    rec = np.sum(E0r * J) * dv / (1j * 2 * np.pi * cfg.freq * physics.MU0)
    assert abs(mr @ Hs - rec) < 1e-12 * abs(rec)


def test_zero_contrast_gives_incident_H():
    cfg = make_config("c1")
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = np.zeros((8, 8, 8, 3, 3))
    src, m = cfg.sources[0]
    E = np.zeros((3, 8, 8, 8), complex)
    H = receivers.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, E, cfg.receivers, src, m)
    H0 = physics.incident_H(np.array(cfg.receivers), src, m, k0)
    assert np.abs(H - H0).max() <= 1e-15 * np.abs(H0).max()
