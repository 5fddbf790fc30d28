"""Pins of oracle/physics.py against things other than itself (CPU, -m "not gpu").

Each test names what fixes the expected value: a paper statement, a textbook limit, an
identity of the Helmholtz operator, or an independent numerical route (finite differences,
quadrature)."""

import json
import os

import numpy as np
import pytest

from oracle import physics

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_wavenumber_branch_and_paper_skin_depth():
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))["skin_depth_section_3_1"]
    k0 = physics.wavenumber(gold["sigma0"], gold["freq_hz"])
    assert k0.real > 0 and k0.imag > 0  # decaying branch
    omega = 2 * np.pi * gold["freq_hz"]
    # k0^2 = i omega mu0 sigma0
    assert abs(k0 ** 2 - 1j * omega * 4e-7 * np.pi * gold["sigma0"]) < 1e-15 * abs(k0) ** 2
    # textbook skin depth sqrt(2 / (omega mu0 sigma)) = 1 / Im k0, and P:253's "approximately 10 m"
    delta = np.sqrt(2.0 / (omega * 4e-7 * np.pi * gold["sigma0"]))
    assert abs(1.0 / k0.imag - delta) < 1e-12 * delta
    assert abs(delta - gold["approx_skin_depth_m"]) < gold["rel_tol"] * gold["approx_skin_depth_m"]


def test_scalar_green_static_limit():
    # k0 -> 0: g -> 1 / (4 pi R)  (Eq. 7)
    k0 = physics.wavenumber(1e-14, 1.0)
    for R in (0.3, 1.0, 2.0):
        assert abs(physics.scalar_green(R, k0) - 1.0 / (4 * np.pi * R)) < 1e-10 / R


def _fd_hessian_g(Rv, k0, step):
    """Central-difference Hessian of the scalar Green's function (independent of green_E)."""
    Hs = np.zeros((3, 3), complex)
    g = lambda v: physics.scalar_green(np.linalg.norm(v), k0)
    for i in range(3):
        for j in range(3):
            ei = np.eye(3)[i] * step
            ej = np.eye(3)[j] * step
            Hs[i, j] = (g(Rv + ei + ej) - g(Rv + ei - ej) - g(Rv - ei + ej) + g(Rv - ei - ej)) / (4 * step * step)
    return Hs


@pytest.mark.parametrize("sigma,freq", [(0.1, 2e6), (1.0, 1e5), (0.5, 4e5)])
def test_green_E_matches_definition_by_finite_differences(sigma, freq):
    """Eq. 5: G^E = (i omega mu0 I + grad grad / sigma0) g, with grad grad g by central FD."""
    rng = np.random.default_rng(7)
    k0 = physics.wavenumber(sigma, freq)
    omega = 2 * np.pi * freq
    for _ in range(6):
        Rv = rng.uniform(-1.5, 1.5, 3)
        Rv *= max(1.0, 0.3 / np.linalg.norm(Rv))
        fd = 1j * omega * physics.MU0 * physics.scalar_green(np.linalg.norm(Rv), k0) * np.eye(3) \
            + _fd_hessian_g(Rv, k0, 1e-4) / sigma
        G = physics.green_E(Rv, k0, sigma)
        assert np.abs(G - fd).max() < 2e-6 * np.abs(G).max()


def test_green_E_trace_symmetry_parity():
    """Tr G^E = 2 i omega mu0 g for R != 0 (since lap g = -k0^2 g); G symmetric; G(-R) = G(R)."""
    rng = np.random.default_rng(3)
    sigma, freq = 0.1, 2e6
    k0 = physics.wavenumber(sigma, freq)
    omega = 2 * np.pi * freq
    for _ in range(10):
        Rv = rng.standard_normal(3)
        G = physics.green_E(Rv, k0, sigma)
        g = physics.scalar_green(np.linalg.norm(Rv), k0)
        assert abs(np.trace(G) - 2j * omega * physics.MU0 * g) < 1e-13 * abs(G).max()
        assert np.abs(G - G.T).max() == 0.0
        assert np.abs(physics.green_E(-Rv, k0, sigma) - G).max() < 1e-15 * abs(G).max()


def test_green_E_static_limit():
    """k0 -> 0: G^E -> (3 Rhat Rhat - I) / (4 pi sigma0 R^3) (electrostatic dipole kernel)."""
    sigma = 0.7
    k0 = physics.wavenumber(sigma, 1e-9)
    Rv = np.array([0.3, -0.4, 1.2])
    R = np.linalg.norm(Rv)
    Rh = Rv / R
    expect = (3 * np.outer(Rh, Rh) - np.eye(3)) / (4 * np.pi * sigma * R ** 3)
    assert np.abs(physics.green_E(Rv, k0, sigma) - expect).max() < 1e-8 * np.abs(expect).max()


@pytest.mark.parametrize("sigma,freq,h", [(0.1, 2e6, 0.1), (1.0, 1e5, 0.25), (0.5, 1e5, 0.2), (0.01, 4e5, 0.25),
                                          (1.0, 4e5, 1.5)])
def test_self_term_against_spherical_quadrature(sigma, freq, h):
    """the singular cell is the integral of Eq. 5 over the equivolume sphere.  Computed
    here by 3-D quadrature (Gauss-Legendre in r and cos(theta), trapezoid in phi) of the
    full tensor G^E, plus the textbook depolarisation term -L/sigma0 with L = I/3 for a
    sphere (the delta-function part of grad grad g that a principal-value integral misses)."""
    k0 = physics.wavenumber(sigma, freq)
    dv = h ** 3
    a = (3 * dv / (4 * np.pi)) ** (1 / 3)
    xr, wr = np.polynomial.legendre.leggauss(40)
    r = 0.5 * a * (xr + 1)
    wr = 0.5 * a * wr
    xc, wc = np.polynomial.legendre.leggauss(8)
    nphi = 8
    phi = 2 * np.pi * np.arange(nphi) / nphi
    total = np.zeros((3, 3), complex)
    for ri, wri in zip(r, wr):
        for ct, wct in zip(xc, wc):
            st = np.sqrt(1 - ct * ct)
            for ph in phi:
                Rv = ri * np.array([st * np.cos(ph), st * np.sin(ph), ct])
                total += physics.green_E(Rv, k0, sigma) * ri * ri * wri * wct * (2 * np.pi / nphi)
    total += -np.eye(3) / (3 * sigma)
    K0 = physics.self_term(k0, sigma, dv)
    assert np.abs(total - K0).max() < 1e-9 * np.abs(K0).max()
    # static limit (S:155 / depolarisation): -I / (3 sigma0)
    K0s = physics.self_term(physics.wavenumber(sigma, 1e-12), sigma, dv)
    assert np.abs(K0s + np.eye(3) / (3 * sigma)).max() < 1e-9 / sigma


def _fd_curl(f, r, step=1e-5):
    J = np.zeros((3, 3), complex)  # J[i, j] = d f_i / d x_j
    for j in range(3):
        e = np.eye(3)[j] * step
        J[:, j] = (f(r + e) - f(r - e)) / (2 * step)
    return np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])


@pytest.mark.parametrize("sigma,freq", [(0.1, 24e3), (1.0, 1e5), (0.1, 2e6)])
def test_incident_fields_curl_consistency(sigma, freq):
    """Eq. 1 away from the source: curl E0 = i omega mu0 H0; checked by central FD."""
    rng = np.random.default_rng(11)
    k0 = physics.wavenumber(sigma, freq)
    omega = 2 * np.pi * freq
    src = np.array([0.1, -0.2, 0.3])
    m = rng.standard_normal(3)
    for _ in range(8):
        r = src + rng.uniform(0.5, 3.0) * rng.standard_normal(3) / np.sqrt(3)
        if np.linalg.norm(r - src) < 0.3:
            continue
        curl = _fd_curl(lambda p: physics.incident_E(p, src, m, k0, freq), r)
        H = physics.incident_H(r, src, m, k0)
        assert np.abs(curl / (1j * omega * physics.MU0) - H).max() < 1e-6 * np.abs(H).max()


def test_incident_static_limits_and_axis():
    """k0 -> 0: axial |H| = m / (2 pi R^3), equatorial |H| = m / (4 pi R^3);
    E0 vanishes on the dipole axis (grad g parallel to m)."""
    k0 = physics.wavenumber(1e-14, 1.0)
    m = np.array([0.0, 0.0, 2.0])
    R = 1.7
    Hax = physics.incident_H(np.array([0, 0, R]), np.zeros(3), m, k0)
    Heq = physics.incident_H(np.array([R, 0, 0]), np.zeros(3), m, k0)
    assert abs(np.linalg.norm(Hax) - 2.0 / (2 * np.pi * R ** 3)) < 1e-9
    assert abs(np.linalg.norm(Heq) - 2.0 / (4 * np.pi * R ** 3)) < 1e-9
    k1 = physics.wavenumber(0.3, 1e5)
    assert np.abs(physics.incident_E(np.array([0, 0, -2.5]), np.zeros(3), m, k1, 1e5)).max() == 0.0
