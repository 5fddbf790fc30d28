"""Pins of the discretisation scale (dv) and of the receiver voltage, against things the
paper and the mathematics fix rather than against the oracle's own formulas (VERDICT r1,
weak #1).

* The discrete kernel K(d) = G^E(d h) dv (Eq. 8) is the midpoint rule of the volume
  integral of Eq. 3.  A uniform contrast source over a block of cells must therefore radiate,
  at cells well outside the block, the continuum volume integral of Eq. 5 over the block,
  computed here by a high-order Gauss rule of the closed-form G^E (itself pinned by finite
  differences in test_oracle_physics).  Dropping or squaring dv changes the result by
  1/dv or dv (10^3 at h = 0.1 m).
* The IE solution of a single cell at low frequency is the static depolarisation of an
  equivolume sphere, E_in = 3 sigma_b / (sigma + 2 sigma_b) E0 (the sign of I - G dsigma).
* h-refinement of one physical body (dense LU at 2^3 / 4^3 / 8^3 cells): the induced current
  dipole converges (differences shrink by a stable factor); with a wrong dv it diverges.
* Receiver voltage (reading R14): Faraday's law (Eq. 1, e^{-i omega t}):
  the loop integral of E around a small coil equals i omega mu0 times the flux of H, so
  ``receivers.voltage(H, m_r)`` with |m_r| = coil area must equal the loop integral of E,
  sign included, for the incident and for the scattered field.
"""

import numpy as np
import pytest

from oracle import physics, operator as op, receivers


def _gauss_cube(center, side, order=6, sub=2):
    """Tensor Gauss-Legendre nodes/weights over an axis-aligned cube (sub^3 sub-cubes)."""
    x, w = np.polynomial.legendre.leggauss(order)
    edges = np.linspace(-side / 2, side / 2, sub + 1)
    pts1, wts1 = [], []
    for a, b in zip(edges[:-1], edges[1:]):
        pts1.append(0.5 * (a + b) + 0.5 * (b - a) * x)
        wts1.append(0.5 * (b - a) * w)
    p1 = np.concatenate(pts1)
    w1 = np.concatenate(wts1)
    Z, Y, X = np.meshgrid(p1, p1, p1, indexing="ij")
    W = w1[:, None, None] * w1[None, :, None] * w1[None, None, :]
    P = np.stack([X, Y, Z], axis=-1).reshape(-1, 3) + np.asarray(center)
    return P, W.ravel()


@pytest.mark.parametrize("sigma_b,freq", [(0.5, 1e5), (0.1, 2e6)])
def test_uniform_block_radiates_the_continuum_volume_integral(sigma_b, freq):
    """scatter() of a uniform J over a 4^3-cell block = integral of G^E over the block (Eq. 3),
    at cells >= 3 block sides away; midpoint-rule error O((h/R)^2) << the 1e3 of a dv error."""
    n, h = (24, 6, 6), 0.1
    nx, ny, nz = n
    hv = (h, h, h)
    k0 = physics.wavenumber(sigma_b, freq)
    rng = np.random.default_rng(11)
    A = rng.standard_normal((3, 3))
    dsig = 0.5 * (A + A.T)  # constant anisotropic contrast inside the block
    ds = np.zeros((nz, ny, nx, 3, 3))
    ds[1:5, 1:5, 0:4] = dsig
    E = np.zeros((3, nz, ny, nx), complex)
    e_in = np.array([1.0, -0.5 + 0.3j, 0.25j])
    E[:, 1:5, 1:5, 0:4] = e_in[:, None, None, None]
    origin = (0.0, 0.0, 0.0)
    s = op.Operator(n, hv, k0, sigma_b, ds).scatter(E)
    J = dsig @ e_in
    # block of cells x in [0,4), y,z in [1,5): faces at -h/2 .. 3.5h
    center = np.array([1.5 * h, 2.5 * h, 2.5 * h])
    P, W = _gauss_cube(center, 4 * h)
    for cx in (14, 18, 23):
        r = np.array([cx * h, 3 * h, 1 * h]) + np.asarray(origin)
        G = physics.green_E(r - P, k0, sigma_b)  # (M, 3, 3)
        ref = np.einsum("m,mpq,q->p", W, G, J)
        got = s[:, 1, 3, cx]
        assert np.linalg.norm(got - ref) < 5e-3 * np.linalg.norm(ref), (cx, got, ref)


def test_single_cell_is_the_static_depolarised_sphere():
    """One cell of conductivity sigma in sigma_b at 1 Hz: E_in = 3 sigma_b/(sigma + 2 sigma_b) E0
    (equivolume-sphere self term, reading R3, with the sign of Eq. 8)."""
    n, h, sigma_b, freq = (1, 1, 1), (0.3, 0.3, 0.3), 0.2, 1.0
    k0 = physics.wavenumber(sigma_b, freq)
    for sig in (0.05, 1.0, 7.0):
        ds = np.full((1, 1, 1, 3, 3), 0.0)
        ds[0, 0, 0] = (sig - sigma_b) * np.eye(3)
        A = op.dense_matrix(n, h, k0, sigma_b, ds)
        E0 = np.array([0.3, -1.0, 0.7], complex)
        E = np.linalg.solve(A, E0)
        expect = 3 * sigma_b / (sig + 2 * sigma_b) * E0
        assert np.abs(E - expect).max() < 1e-6 * np.abs(E0).max()


def test_h_refinement_of_one_body_converges():
    """A 0.5 m cube (sigma = 3 sigma_b, anisotropic) in a uniform-ish incident field, discretised
    at 2^3, 4^3, 8^3 cells and solved by dense LU: the induced current dipole p = sum J dv
    converges with a stable observed order (differences shrink >= 1.6x per halving)."""
    sigma_b, freq, side = 0.5, 1e4, 0.5
    k0 = physics.wavenumber(sigma_b, freq)
    sig = np.array([[1.5, 0.2, 0.1], [0.2, 1.2, -0.1], [0.1, -0.1, 1.8]])
    src, m = np.array([0.0, 0.0, 3.0]), np.array([1.0, 0.3, 0.2])
    ps = []
    for nc in (2, 4, 8):
        h = side / nc
        n = (nc, nc, nc)
        origin = tuple([-(nc - 1) / 2 * h] * 3)
        ds = np.broadcast_to(sig - sigma_b * np.eye(3), (nc, nc, nc, 3, 3)).copy()
        pts = physics.centroids(n, (h, h, h), origin)
        E0 = np.moveaxis(physics.incident_E(pts, src, m, k0, freq), -1, 0)
        A = op.dense_matrix(n, (h, h, h), k0, sigma_b, ds)
        E = np.linalg.solve(A, E0.ravel()).reshape(E0.shape)
        J = op.contrast_source(ds, E)
        ps.append(J.reshape(3, -1).sum(axis=1) * h ** 3)
    d1 = np.linalg.norm(ps[1] - ps[0])
    d2 = np.linalg.norm(ps[2] - ps[1])
    assert d2 < d1 / 1.6, (d1, d2)
    assert d2 < 0.05 * np.linalg.norm(ps[2])


def _loop(center, normal, b, npts=256):
    """Points and tangent vectors dl of a circle of radius b, orientation by the right-hand rule."""
    nrm = np.asarray(normal, float) / np.linalg.norm(normal)
    a = np.cross(nrm, [1.0, 0.0, 0.0])
    if np.linalg.norm(a) < 0.1:
        a = np.cross(nrm, [0.0, 1.0, 0.0])
    a /= np.linalg.norm(a)
    c = np.cross(nrm, a)
    t = 2 * np.pi * np.arange(npts) / npts
    P = center + b * (np.cos(t)[:, None] * a + np.sin(t)[:, None] * c)
    dl = b * (-np.sin(t)[:, None] * a + np.cos(t)[:, None] * c) * (2 * np.pi / npts)
    return P, dl


def _disk(center, normal, b, nr=24, nt=64):
    nrm = np.asarray(normal, float) / np.linalg.norm(normal)
    a = np.cross(nrm, [1.0, 0.0, 0.0])
    if np.linalg.norm(a) < 0.1:
        a = np.cross(nrm, [0.0, 1.0, 0.0])
    a /= np.linalg.norm(a)
    c = np.cross(nrm, a)
    x, w = np.polynomial.legendre.leggauss(nr)
    r = 0.5 * b * (x + 1)
    wr = 0.5 * b * w * r
    t = 2 * np.pi * np.arange(nt) / nt
    P = center + r[:, None, None] * (np.cos(t)[None, :, None] * a + np.sin(t)[None, :, None] * c)
    W = wr[:, None] * np.full(nt, 2 * np.pi / nt)[None, :]
    return P.reshape(-1, 3), W.ravel()


@pytest.mark.parametrize("normal", [(0, 0, 1), (1, 0, 0), (0.3, -0.8, 0.5)])
def test_voltage_is_faradays_loop_integral_of_the_incident_field(normal):
    """EMF = loop integral of E0 = i omega mu0 * flux of H0 (Eq. 1); for a small coil of area A
    with normal n, voltage(H0(r), A n) equals it (sign included), and Stokes holds exactly."""
    sigma_b, freq = 0.3, 4e5
    k0 = physics.wavenumber(sigma_b, freq)
    src, m = np.array([0.1, -0.2, 0.0]), np.array([0.2, 0.5, 1.0])
    r = np.array([0.4, 0.3, 1.1])
    n_hat = np.asarray(normal, float) / np.linalg.norm(normal)
    # exact Stokes on a finite disk (b = 0.2 m)
    b = 0.2
    P, dl = _loop(r, n_hat, b)
    emf = np.sum(physics.incident_E(P, src, m, k0, freq) * dl)
    Pd, Wd = _disk(r, n_hat, b)
    flux = np.sum(Wd * (physics.incident_H(Pd, src, m, k0) @ n_hat))
    omega = physics.omega_of(freq)
    assert abs(emf - 1j * omega * physics.MU0 * flux) < 1e-9 * abs(emf)
    # small coil: the receiver voltage of a coil of area A along n
    b = 1e-3
    P, dl = _loop(r, n_hat, b)
    emf = np.sum(physics.incident_E(P, src, m, k0, freq) * dl)
    v = receivers.voltage(physics.incident_H(r, src, m, k0), np.pi * b * b * n_hat, freq)
    assert abs(v - emf) < 1e-5 * abs(emf)
    # a flipped iωμ0 sign would give the conjugate-like value; make sure it is distinguishable
    assert abs(-np.conj(v) - emf) > 1e-2 * abs(emf)


def test_scattered_receiver_field_obeys_faraday():
    """The scattered H of receivers.receiver_H (Eq. 4 with Eq. 6) and the scattered E radiated by
    the same contrast currents (Eq. 3 at an off-grid point, midpoint rule as Eq. 8) satisfy
    Faraday's law around a coil outside the body: loop integral of E_s = i omega mu0 flux(H_s)."""
    n, h, sigma_b, freq = (4, 4, 4), (0.25, 0.25, 0.25), 0.5, 2e5
    k0 = physics.wavenumber(sigma_b, freq)
    origin = (-0.375, -0.375, -0.375)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((4, 4, 4, 3, 3))
    ds = 0.5 * (A + np.swapaxes(A, -1, -2)) + 1.5 * np.eye(3)
    src, m = np.array([0.0, 0.0, 1.5]), np.array([0.0, 0.0, 1.0])
    pts = physics.centroids(n, h, origin)
    E0 = np.moveaxis(physics.incident_E(pts, src, m, k0, freq), -1, 0)
    E = np.linalg.solve(op.dense_matrix(n, h, k0, sigma_b, ds), E0.ravel()).reshape(E0.shape)
    J = np.moveaxis(op.contrast_source(ds, E), 0, -1).reshape(-1, 3)
    rc = pts.reshape(-1, 3)
    dv = h[0] * h[1] * h[2]
    # the scattered E at a cell centroid from this formula equals the operator's scatter()
    Es_grid = op.Operator(n, h, k0, sigma_b, ds).scatter(E)
    c = (3, 1, 2)
    r_c = pts[c[2], c[1], c[0]]
    Rv = r_c - rc
    mask = np.linalg.norm(Rv, axis=1) > 0
    es = np.einsum("mpq,mq->p", physics.green_E(Rv[mask], k0, sigma_b), J[mask]) * dv \
        + physics.self_term(k0, sigma_b, dv) @ J[~mask][0]
    assert np.abs(es - Es_grid[:, c[2], c[1], c[0]]).max() < 1e-12 * np.abs(es).max()

    def E_s(P):
        return np.einsum("kmpq,mq->kp", physics.green_E(P[:, None, :] - rc[None], k0, sigma_b), J) * dv

    r, n_hat, b = np.array([0.2, -0.1, 1.2]), np.array([0.6, 0.0, 0.8]), 0.15
    P, dl = _loop(r, n_hat, b, npts=128)
    emf = np.sum(E_s(P) * dl)
    Pd, Wd = _disk(r, n_hat, b, nr=16, nt=48)
    Hs = receivers.receiver_H(n, h, origin, k0, sigma_b, ds, E, Pd, src, m) - physics.incident_H(Pd, src, m, k0)
    flux = np.sum(Wd * (Hs @ n_hat))
    omega = physics.omega_of(freq)
    assert abs(emf - 1j * omega * physics.MU0 * flux) < 1e-8 * abs(emf)
