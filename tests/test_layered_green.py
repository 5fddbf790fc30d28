"""Pins of the layered-background generator ie_workloads/layered_green.py (the host tables and
incident fields BASELINE.json c3/c4 name as input data for both paths; R21).

What fixes a layered Green's function independently of the code that computes it:
  * equal layers: every reflection vanishes and the transmitted-path machinery (1-D Green's
    functions, TE/TM assembly, Hankel quadrature, angular factors) must reproduce the closed-form
    homogeneous Eq. 5 / incident fields of the oracle (oracle/physics.py), above AND below the
    source (the latter goes through the mirrored medium);
  * Maxwell's interface conditions: tangential E, normal current sigma E_z and (mu = mu0) all of H
    are continuous across every interface;
  * Faraday in the layered medium: curl E0 = i omega mu0 H0 off the source;
  * reciprocity of a reciprocal medium: G_pq(r, r') = G_qp(r', r) (in an ASYMMETRIC three-layer
    medium, where the observer-below branch is computed through a different mirrored medium),
    m_r . H^{m_s}(r_r) = m_s . H^{m_r}(r_s);
  * the omega -> 0 limit: G^E -> -grad grad'^T Phi with Phi the textbook image series of a point
    current source in a conducting slab between two half-spaces;
  * the table: equal-layer table = the oracle's homogeneous (degenerate) table; the stored
    quadrant obeys the signed reciprocity T_pq(D; k, k') = s_p s_q T_qp(D; k', k) with the mirror
    signs of reading R18; interpolated entries equal direct point evaluation.
"""

import numpy as np
import pytest

from ie_workloads import layered_green as lg
from oracle import physics, layered as lay

SX = np.array([-1.0, 1.0, 1.0])
SY = np.array([1.0, -1.0, 1.0])


@pytest.mark.parametrize("layers,zi", [((0.3, 0.3), (0.1,)), ((0.3, 0.3, 0.3), (-0.3, 0.4))])
def test_equal_layers_reproduce_the_homogeneous_dyadic(layers, zi):
    sig, f = 0.3, 4e5
    med = lg.Medium(layers, zi, f)
    k0 = physics.wavenumber(sig, f)
    pairs = [([0.5, 0.2, 0.6], [0.0, 0.0, -0.5]), ([0.5, -0.7, -0.6], [0.1, 0.3, 0.8]),
             ([0.0, 0.0, 0.7], [0.0, 0.0, -0.4]), ([2.5, 1.0, 0.9], [0.0, 0.0, -0.5]),
             ([-1.2, 0.4, 0.45], [0.3, -0.2, 0.35])]
    for ro, rs in pairs:
        ro, rs = np.array(ro), np.array(rs)
        G = lg.dyadic_at(med, ro[None], rs[None])[0]
        ref = physics.green_E(ro - rs, k0, sig)
        assert np.abs(G - ref).max() < 1e-12 * np.abs(ref).max()


def test_equal_layers_reproduce_the_homogeneous_incident_fields():
    sig, f = 0.3, 4e5
    med = lg.Medium((sig, sig, sig), (-0.3, 0.4), f)
    k0 = physics.wavenumber(sig, f)
    rng = np.random.default_rng(0)
    src = np.array([0.05, -0.1, -0.02])
    pts = rng.uniform(-2, 2, size=(40, 3))
    pts[:, 2] = np.round(pts[:, 2] * 4) / 4 + 0.125
    mom = np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], [0.3, -0.5, 0.8]])
    E = lg.incident_E_layered(med, pts, src, mom)
    H = lg.incident_H_layered(med, pts[:6], src, mom)
    for t, m in enumerate(mom):
        Er = physics.incident_E(pts, src, m, k0, f)
        Hr = physics.incident_H(pts[:6], src, m, k0)
        assert np.abs(E[t] - Er).max() < 1e-10 * np.abs(Er).max()
        assert np.abs(H[t] - Hr).max() < 1e-12 * np.abs(Hr).max()


MED3 = dict(sigma=(1.0, 0.01, 0.3), zi=(-4.0, 3.0))  # asymmetric three-layer medium


def _med3(f=4e5):
    return lg.Medium(MED3["sigma"], MED3["zi"], f)


@pytest.mark.parametrize("zi", [3.0, -4.0])
def test_dyadic_interface_conditions(zi):
    """Tangential E and normal current continuous across the interface: the jump at +-eps
    vanishes linearly with eps (smooth fields on each side)."""
    med = _med3()
    for rs in (np.array([0.3, -0.2, 2.1]), np.array([-0.5, 0.4, -6.0]), np.array([0.2, 0.1, 5.0])):
        d = []
        for eps in (1e-6, 1e-8):
            a = lg.dyadic_at(med, np.array([[1.1, 0.7, zi + eps]]), rs[None])[0]
            b = lg.dyadic_at(med, np.array([[1.1, 0.7, zi - eps]]), rs[None])[0]
            sa, sb = med.sigma_at(zi + eps), med.sigma_at(zi - eps)
            scale = np.abs(a).max()
            d.append((np.abs(a[:2] - b[:2]).max() / scale, np.abs(sa * a[2] - sb * b[2]).max() / (sa * np.abs(a[2]).max())))
        # the differences shrink with eps (x 1e-2 here): O(eps) gradients, no jump
        assert d[1][0] < 0.02 * d[0][0] + 1e-10 and d[1][1] < 0.02 * d[0][1] + 1e-10, d


@pytest.mark.parametrize("zi", [3.0, -4.0])
def test_incident_field_interface_conditions(zi):
    med = _med3()
    rs = np.array([0.3, -0.2, 1.1])
    mom = np.array([[0.3, -0.5, 0.8], [1.0, 0.0, 0.0]])
    d = []
    for eps in (1e-6, 1e-8):
        pa = np.array([[1.1, 0.7, zi + eps], [-2.0, 0.3, zi + eps]])
        pb = np.array([[1.1, 0.7, zi - eps], [-2.0, 0.3, zi - eps]])
        Ea = lg.incident_E_layered(med, pa, rs, mom, rho_interp=False)
        Eb = lg.incident_E_layered(med, pb, rs, mom, rho_interp=False)
        Ha = lg.incident_H_layered(med, pa, rs, mom)
        Hb = lg.incident_H_layered(med, pb, rs, mom)
        sa, sb = med.sigma_at(zi + eps), med.sigma_at(zi - eps)
        d.append((np.abs(Ea[..., :2] - Eb[..., :2]).max() / np.abs(Ea).max(),
                  np.abs(sa * Ea[..., 2] - sb * Eb[..., 2]).max() / (sa * np.abs(Ea[..., 2]).max()),
                  np.abs(Ha - Hb).max() / np.abs(Ha).max()))
    for a, b in zip(d[1], d[0]):  # O(eps) differences: no jump
        assert a < 0.02 * b + 1e-10, d


def test_incident_fields_obey_faraday_in_the_layered_medium():
    med = _med3()
    rs = np.array([0.3, -0.2, 2.1])
    mom = np.array([[0.3, -0.5, 0.8]])
    for r0 in (np.array([1.3, -0.4, -4.6]), np.array([0.5, 0.9, 2.6]), np.array([-1.0, 0.2, 4.0])):
        d = 1e-4

        def E(p):
            return lg.incident_E_layered(med, np.atleast_2d(p), rs, mom, rho_interp=False)[0, 0]

        J = np.zeros((3, 3), complex)
        for a in range(3):
            e = np.zeros(3)
            e[a] = d
            J[:, a] = (E(r0 + e) - E(r0 - e)) / (2 * d)
        curl = np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])
        H = lg.incident_H_layered(med, r0[None], rs, mom)[0, 0]
        assert np.abs(curl - 1j * med.omega * lg.MU0 * H).max() < 1e-6 * np.abs(curl).max()


def test_reciprocity_in_an_asymmetric_medium():
    med = _med3()
    pts = [np.array(p) for p in ([1.0, 0.5, -5.0], [0.4, -1.2, 6.3], [2.0, 1.0, 2.5], [0.0, 0.0, 1.5],
                                 [3.0, -2.0, -7.0], [0.1, 0.2, -6.0], [0.0, 0.3, 5.0])]
    for i, a in enumerate(pts):
        for b in pts[i + 1:]:
            G1 = lg.dyadic_at(med, a[None], b[None])[0]
            G2 = lg.dyadic_at(med, b[None], a[None])[0]
            assert np.abs(G1 - G2.T).max() < 1e-12 * np.abs(G1).max()
    rs, ms = np.array([0.3, -0.2, 2.1]), np.array([0.3, -0.5, 0.8])
    for rr, mr in ((np.array([0.5, 0.9, -4.8]), np.array([0.2, 1.0, -0.4])),
                   (np.array([-1.5, 0.2, 3.7]), np.array([1.0, 0.0, 0.3]))):
        a = mr @ lg.incident_H_layered(med, rr[None], rs, ms[None])[0, 0]
        b = ms @ lg.incident_H_layered(med, rs[None], rr, mr[None])[0, 0]
        assert abs(a - b) < 1e-12 * abs(a)


def test_mirror_parities():
    """G_pq(-x, y) = sx_p sx_q G_pq(x, y), G_pq(x, -y) = sy_p sy_q G_pq(x, y) (horizontally layered
    isotropic medium; the storage rule of reading R18)."""
    med = _med3()
    rs = np.array([0.0, 0.0, 2.1])
    for ro in (np.array([1.1, 0.6, -5.0]), np.array([0.7, 1.3, 2.6])):
        G = lg.dyadic_at(med, ro[None], rs[None])[0]
        Gx = lg.dyadic_at(med, (ro * [-1, 1, 1])[None], rs[None])[0]
        Gy = lg.dyadic_at(med, (ro * [1, -1, 1])[None], rs[None])[0]
        assert np.abs(Gx - np.outer(SX, SX) * G).max() < 1e-14 * np.abs(G).max()
        assert np.abs(Gy - np.outer(SY, SY) * G).max() < 1e-14 * np.abs(G).max()


def test_static_limit_is_the_image_series():
    """omega -> 0: G^E = -grad grad'^T Phi, Phi = (1/4 pi s2)[1/R + sum_n (pt pb)^n (pt/R_t,n + pb/R_b,n)
    + sum_{n>=1} (pt pb)^n (1/R_+n + 1/R_-n)], pt = (s2-s3)/(s2+s3), pb = (s2-s1)/(s2+s1), images at
    2zt - z' + 2nd, 2zb - z' - 2nd, z' +- 2nd (source and observer in the slab)."""
    s1, s2, s3 = MED3["sigma"]
    zb, zt = MED3["zi"]
    d = zt - zb
    med = lg.Medium((s1, s2, s3), (zb, zt), 1e-4)
    pt, pb = (s2 - s3) / (s2 + s3), (s2 - s1) / (s2 + s1)

    def G_static(ro, rsrc):
        zp = rsrc[2]
        terms = [(1.0, zp, 1.0)]
        for n in range(0, 4000):
            f = (pt * pb) ** n
            terms.append((f * pt, 2 * zt - zp + 2 * n * d, -1.0))
            terms.append((f * pb, 2 * zb - zp - 2 * n * d, -1.0))
            if n >= 1:
                terms.append((f, zp + 2 * n * d, 1.0))
                terms.append((f, zp - 2 * n * d, 1.0))
        out = np.zeros((3, 3))
        for c, zimg, sgn in terms:
            R = ro - np.array([rsrc[0], rsrc[1], zimg])
            Rn = np.linalg.norm(R)
            Hm = (3 * np.outer(R, R) - Rn ** 2 * np.eye(3)) / Rn ** 5  # grad grad (1/R)
            out -= c * Hm * np.array([1.0, 1.0, sgn])[None, :]  # grad grad'^T (1/R)
        return -out / (4 * np.pi * s2)

    rsrc = np.array([0.1, -0.3, 1.0])
    for ro in ([1.5, 0.5, -2.0], [0.3, 2.2, 2.5], [4.0, 1.0, 0.0]):
        ro = np.array(ro)
        G = lg.dyadic_at(med, ro[None], rsrc[None])[0]
        Gs = G_static(ro, rsrc)
        assert np.abs(G - Gs).max() < 1e-7 * np.abs(Gs).max()


def test_equal_layer_table_is_the_homogeneous_table():
    n, h, sig, f = (6, 5, 8), (0.25, 0.25, 0.25), 0.4, 4e5
    origin = tuple(-(a - 1) / 2 * 0.25 for a in n)
    ref = lay.homogeneous_table(n, h, physics.wavenumber(sig, f), sig)
    # one layer: closed form only
    T1 = lg.layered_table(lg.Medium((sig,), (), f), n, h, origin)
    assert np.abs(T1 - ref).max() < 1e-14 * np.abs(ref).max()
    # equal layers with interfaces: the cross-interface pairs come out of the Hankel quadrature
    T = lg.layered_table(lg.Medium((sig, sig, sig), (-0.5, 0.5), f), n, h, origin)
    assert np.abs(T - ref).max() < 1e-10 * np.abs(ref).max()


@pytest.fixture(scope="module")
def phys_table():
    n, h = (8, 6, 16), (0.25, 0.25, 0.25)
    origin = tuple(-(a - 1) / 2 * 0.25 for a in n)
    med = lg.Medium((1.0, 0.01, 0.3), (-1.0, 0.5), 4e5)
    return med, n, h, origin, lg.layered_table(med, n, h, origin)


def test_table_signed_reciprocity(phys_table):
    med, n, h, origin, T = phys_table
    s = np.outer(SX * SY, SX * SY)  # (p, q)
    Tt = np.swapaxes(np.swapaxes(T, 0, 1), 2, 3)  # T_qp(k', k)
    assert np.abs(T - s[:, :, None, None, None, None] * Tt).max() < 1e-12 * np.abs(T).max()


def test_table_entries_equal_direct_evaluation(phys_table):
    med, n, h, origin, T = phys_table
    nx, ny, nz = n
    z = origin[2] + h[2] * np.arange(nz)
    dv = h[0] * h[1] * h[2]
    rng = np.random.default_rng(3)
    for _ in range(25):
        di, dj, k, kp = rng.integers(0, nx), rng.integers(0, ny), rng.integers(0, nz), rng.integers(0, nz)
        if di == 0 and dj == 0 and k == kp:
            continue
        ro = np.array([di * h[0], dj * h[1], z[k]])
        rs = np.array([0.0, 0.0, z[kp]])
        G = lg.dyadic_at(med, ro[None], rs[None])[0] * dv
        assert np.abs(G - T[:, :, k, kp, dj, di]).max() < 1e-9 * np.abs(G).max()


def test_centroid_on_an_interface_is_rejected():
    med = lg.Medium((1.0, 0.1), (0.0,), 1e5)
    with pytest.raises(AssertionError):
        lg.layered_table(med, (2, 2, 4), (0.25, 0.25, 0.25), (0.0, 0.0, -0.25))


def test_grid_incident_field_equals_point_evaluation():
    """incident_E_layered_grid (the one the layered inputs use: radial functions per depth,
    interpolated to the (x, y) columns) equals the point evaluation without interpolation, for
    moments with every component, sources in each layer and next to an interface; and with equal
    layers it equals the oracle's homogeneous incident field."""
    med = _med3()
    x = -1.375 + 0.25 * np.arange(12)
    y = -0.875 + 0.25 * np.arange(8)
    z = np.array([-6.125, -4.125, -3.875, 0.125, 2.875, 3.125, 5.375])
    moms = np.array([[0.3, -0.5, 0.8], [1.0, 0.2, -0.4]])
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    P = np.stack([X, Y, Z], -1).reshape(-1, 3)
    for src in (np.array([0.05, 0.1, 0.4]), np.array([-0.3, 0.2, -5.0]), np.array([0.1, -0.05, 2.98]),
                np.array([0.2, 0.3, 4.6])):
        Eg = lg.incident_E_layered_grid(med, x, y, z, src, moms)  # (2, 3, nz, ny, nx)
        Ep = lg.incident_E_layered(med, P, src, moms, rho_interp=False)  # (2, P, 3)
        Ep = np.moveaxis(Ep.reshape(2, len(z), len(y), len(x), 3), -1, 1)
        assert np.abs(Eg - Ep).max() < 1e-9 * np.abs(Ep).max()
    sig, f = 0.3, 4e5
    med1 = lg.Medium((sig, sig), (0.3,), f)
    src = np.array([0.05, 0.1, -0.2])
    Eg = lg.incident_E_layered_grid(med1, x, y, z * 0.1, src, moms)
    k0 = physics.wavenumber(sig, f)
    Z, Y, X = np.meshgrid(z * 0.1, y, x, indexing="ij")
    for t, m in enumerate(moms):
        ref = np.moveaxis(physics.incident_E(np.stack([X, Y, Z], -1), src, m, k0, f), -1, 0)
        assert np.abs(Eg[t] - ref).max() < 1e-10 * np.abs(ref).max()
