"""Green's functions of a horizontally layered, isotropic conducting background -- the host
generator of the layered tables and incident fields that BASELINE.json's c3/c4 name as
INPUT DATA for both paths ("Layered Green's-tensor tables are precomputed on the host as
input data for both paths").  Both the CUDA path and the oracle consume its output bytes;
neither implements it.  The paper's own background is homogeneous; this extends it.

Physics (quasi-static, e^{-i omega t}, mu = mu0 everywhere, Eq. 1-2 of P:34-41 with a
z-dependent sigma(z)): curl E = i omega mu0 (H + M), curl H = sigma E + J.

Spectral (horizontal Fourier) decomposition.  For a horizontal wavevector (kx, ky),
k = |(kx, ky)|, with the rotated frame u = (kx, ky)/k, v = z x u, the fields split into a
TE set (E_v, H_u, H_z) and a TM set (E_u, E_z, H_v), each governed by a 1-D problem
    d/dz (a dG/dz) - a u_j^2 G = -delta(z - z'),   u_j = sqrt(k^2 - k_j^2), k_j^2 = i omega mu0 sigma_j,
with a = 1 (TE) or 1/sigma (TM), G and a dG/dz continuous across interfaces, decaying at
+-infinity.  In layer j the solutions are e^{+-u_j z}; the 1-D Green's function is built from
generalised reflection coefficients (admittances Y_j = a_j u_j):
    source layer m, secondary part:  (M/2Y_m)[Rup e^{-u(zt-z)}e^{-u(zt-z')} + Rdn e^{-u(z-zb)}e^{-u(z'-zb)}
                                     + Rup Rdn e^{-ud}(e^{-u(zt-z)}e^{-u(z'-zb)} + e^{-u(z-zb)}e^{-u(zt-z')})],
                                     M = 1/(1 - Rup Rdn e^{-2ud});
    observer layer n above m:        (1/2Y_m) M_m [T(z') + Rdn_m e_m B(z')] prod_j(tau_j e_j) [B(z) + Rup_n e_n T(z)]
and the observer-below case is the same formula in the z-mirrored medium (so 1-D reciprocity
G(z,z') = G(z',z) is a check, not a construction).  Every exponent is a negative distance.

Electric dyadic for an electric current source p at (0,0,z') (derived from the TE/TM
equations above):
    E_u = A p_u + i k B p_z,  E_z = -i k C p_u + k^2 D p_z,  E_v = T p_v,
    A = d_z d_z' G_TM/(s s'),  B = d_z G_TM/(s s'),  C = d_z' G_TM/(s s'),  D = G_TM/(s s'),  T = i omega mu0 G_TE,
and the horizontal inverse transform gives, with (x, y) = rho (cos phi, sin phi),
    G_xx = P0 - P2 cos2phi,  G_yy = P0 + P2 cos2phi,  G_xy = G_yx = -P2 sin2phi,
    G_xz = -Q1 cos phi,  G_yz = -Q1 sin phi,  G_zx = R1 cos phi,  G_zy = R1 sin phi,  G_zz = Z0,
    P0 = (1/4pi) int (A+T) J0 k dk,  P2 = (1/4pi) int (A-T) J2 k dk,
    Q1 = (1/2pi) int B J1 k^2 dk,  R1 = (1/2pi) int C J1 k^2 dk,  Z0 = (1/2pi) int D J0 k^3 dk.
For z, z' in the same layer the primary part is the homogeneous G^E of Eq. 5 with that
layer's sigma (closed form; the equivolume-ball self term of reading R3 at r = r'), and only
the secondary part goes through the Hankel integrals, which then decay like e^{-k zeta} with
zeta >= the distance to the interfaces (>= h for cell centroids, as cells never straddle an
interface).

Magnetic dipole m at r_s (transmitters, receiver dipoles): E_v = i omega mu0 [-m_u d_zs G_TE
- i k m_z G_TE], E_u = -i omega mu0 (m_v/s) d_z G_TM, E_z = i omega mu0 (i k m_v/s) G_TM, and
H_u = m_u d_z d_zs G_TE + i k m_z d_z G_TE, H_z = -i k m_u d_zs G_TE + k^2 m_z G_TE,
H_v = i omega mu0 m_v G_TM (off the source).

Quadrature: composite Gauss-Legendre in k on [0, kmax], kmax = 38/zeta_min of the block of
(z, z') pairs at hand (the integrand's envelope e^{-k zeta} k^3 is then < 1e-12 of its
integral), panels of at most half a period of J_n(k rho_max) of the radial band.  Radial
dependence: the radial functions are computed on piecewise Chebyshev-Lobatto nodes in rho
(segments [0,h],[h,2h],[2h,4h],[4h,8h] then 2 m) and interpolated barycentrically to the
lattice offsets (accuracy checked against direct evaluation in tests).

Readings (R21): midpoint rule off the self cell, as Eq. 8 / R3 for the homogeneous
kernel; the self cell takes the homogeneous ball term of its layer plus the (smooth)
secondary part at the centroid; displacement currents dropped as in the paper.
"""

import numpy as np
from scipy import special

MU0 = 4e-7 * np.pi
_GL_ORDER = 8
_ZETA_CUT = 38.0


# ------------------------------------------------------------------------------- medium

class Medium:
    """Horizontally layered isotropic background: sigma[j] of layer j (bottom -> top) and the
    ascending interface depths z_iface[j] between layers j and j+1."""

    def __init__(self, sigma, z_iface, freq):
        self.sigma = np.asarray(sigma, np.float64).ravel()
        self.zi = np.asarray(z_iface, np.float64).ravel()
        assert len(self.zi) == len(self.sigma) - 1 and np.all(np.diff(self.zi) > 0)
        assert np.all(self.sigma > 0)
        self.L = len(self.sigma)
        self.freq = float(freq)
        self.omega = 2.0 * np.pi * self.freq
        self.k2 = 1j * self.omega * MU0 * self.sigma

    def layer_of(self, z):
        return np.searchsorted(self.zi, np.asarray(z, np.float64), side="right")

    def zb(self, j):
        return self.zi[j - 1] if j > 0 else -np.inf

    def zt(self, j):
        return self.zi[j] if j < self.L - 1 else np.inf

    def flipped(self):
        return Medium(self.sigma[::-1], -self.zi[::-1], self.freq)

    def sigma_at(self, z):
        return self.sigma[self.layer_of(z)]

    def wavenumber(self, j):
        k = np.sqrt(self.k2[j])
        return complex(k)


# ----------------------------------------------------------------- 1-D Green's function

class Spectral1D:
    """Reflection/transmission data of the TE and TM 1-D problems on a set of wavenumbers k."""

    def __init__(self, med, k):
        self.med = med
        self.k = np.asarray(k, np.float64)
        L = med.L
        self.u = np.sqrt(self.k[:, None] ** 2 - med.k2[None, :])  # principal: Re u > 0
        d = np.array([med.zt(j) - med.zb(j) for j in range(L)])
        with np.errstate(over="ignore", invalid="ignore"):
            self.e = np.where(np.isfinite(d)[None, :], np.exp(-self.u * np.where(np.isfinite(d), d, 0.0)[None, :]), 0.0)
        self.modes = {}
        for mode, a in (("TE", np.ones(L)), ("TM", 1.0 / med.sigma)):
            Y = a[None, :] * self.u
            Rup = np.zeros_like(Y)
            Rdn = np.zeros_like(Y)
            for j in range(L - 2, -1, -1):
                rho = Rup[:, j + 1] * self.e[:, j + 1] ** 2
                num = (1 + rho) * Y[:, j] - (1 - rho) * Y[:, j + 1]
                den = (1 + rho) * Y[:, j] + (1 - rho) * Y[:, j + 1]
                Rup[:, j] = num / den
            for j in range(1, L):
                rho = Rdn[:, j - 1] * self.e[:, j - 1] ** 2
                num = (1 + rho) * Y[:, j] - (1 - rho) * Y[:, j - 1]
                den = (1 + rho) * Y[:, j] + (1 - rho) * Y[:, j - 1]
                Rdn[:, j] = num / den
            M = 1.0 / (1.0 - Rup * Rdn * self.e ** 2)
            self.modes[mode] = (Y, Rup, Rdn, M)

    def terms(self, mode, n, m):
        """Secondary (n == m) or full (n != m) 1-D Green's function of observer layer n and
        source layer m as separable terms [(coef(Q), kind_z, kind_zp)], kinds 'T' = e^{-u(zt-z)},
        'B' = e^{-u(z-zb)} of the observer (z) / source (z') layer."""
        if n < m:
            return None  # handled by the caller through the mirrored medium
        Y, Rup, Rdn, M = self.modes[mode]
        e = self.e
        L = self.med.L
        out = []
        if n == m:
            c = M[:, m] / (2 * Y[:, m])
            if m < L - 1:
                out.append((c * Rup[:, m], "T", "T"))
            if m > 0:
                out.append((c * Rdn[:, m], "B", "B"))
            if 0 < m < L - 1:
                x = c * Rup[:, m] * Rdn[:, m] * e[:, m]
                out.append((x, "T", "B"))
                out.append((x, "B", "T"))
            return out
        P = M[:, m] / (2 * Y[:, m])
        for j in range(m + 1, n + 1):
            rho = Rup[:, j] * e[:, j] ** 2
            tau = 2 * Y[:, j - 1] / (Y[:, j - 1] * (1 + rho) + Y[:, j] * (1 - rho))
            P = P * tau
            if j < n:
                P = P * e[:, j]
        src = [(np.ones_like(P), "T")]
        if m > 0:
            src.append((Rdn[:, m] * e[:, m], "B"))
        obs = [(np.ones_like(P), "B")]
        if n < L - 1:
            obs.append((Rup[:, n] * e[:, n], "T"))
        for co, ko in obs:
            for cs, ks in src:
                out.append((P * co * cs, ko, ks))
        return out


def _pair_terms(med, k, n, m, cache=None):
    """{mode: [(coef, kind_z, kind_zp)]} for observer layer n, source layer m, in ORIGINAL
    coordinates (observer-below through the mirrored medium with T <-> B swapped)."""
    swap = {"T": "B", "B": "T"}
    if n >= m:
        sp = Spectral1D(med, k) if cache is None else cache[0]
        return {mode: sp.terms(mode, n, m) for mode in ("TE", "TM")}
    L = med.L
    sp = Spectral1D(med.flipped(), k) if cache is None else cache[1]
    return {mode: [(c, swap[a], swap[b]) for c, a, b in sp.terms(mode, L - 1 - n, L - 1 - m)] for mode in ("TE", "TM")}


def _factor(med, u_col, j, kind, z):
    """e^{-u_j alpha(z)} (Q, nz), alpha = zt - z ('T') or z - zb ('B') (its d/dz factor is +u_j for
    'T' and -u_j for 'B', applied by the callers)."""
    z = np.asarray(z, np.float64)
    a = (med.zt(j) - z) if kind == "T" else (z - med.zb(j))
    assert np.all(a >= 0) and np.all(np.isfinite(a))
    return np.exp(-u_col[:, None] * a[None, :])


def _alpha(med, j, kind, z):
    z = np.asarray(z, np.float64)
    return (med.zt(j) - z) if kind == "T" else (z - med.zb(j))


# --------------------------------------------------------------------------- quadrature

def _kim(med):
    """Smallest Im k_j over the layers (1 / the largest skin depth)."""
    return float(np.min(np.sqrt(med.k2).imag))


def gl_nodes(kmax, width, order=_GL_ORDER, zeta_max=None, kim_min=None):
    """Composite Gauss-Legendre nodes/weights on [0, kmax].  Panels are at most ``width`` (half a
    period of J_n(k rho_max)) and graded near k = 0 so that every prefix [0, 38/zeta] a block of
    decay rate zeta uses has panels <= 4/zeta (the e^{-k zeta} envelope is then resolved by the
    8-point rule to ~1e-14), and panels near the branch points k = +-k_j of u_j (at distance
    Im k_j = 1/skin depth from the real axis) stay below 0.6 Im k_j:
    width(k) = min(width, max(0.1 k, w0)), w0 = min(width, 4/zeta_max, 0.6 min_j Im k_j)."""
    x, w = np.polynomial.legendre.leggauss(order)
    w0 = width if zeta_max is None else min(width, 4.0 / zeta_max)
    if kim_min is not None:
        w0 = min(w0, 0.6 * kim_min)
    edges = [0.0]
    while edges[-1] < kmax:
        edges.append(min(kmax, edges[-1] + max(w0, min(width, 0.1 * edges[-1]))))
    edges = np.array(edges)
    a, b = edges[:-1, None], edges[1:, None]
    k = (0.5 * (a + b) + 0.5 * (b - a) * x[None, :]).ravel()
    wk = (0.5 * (b - a) * w[None, :]).ravel()
    return k, wk


def radial_nodes(rho_max, h, seg_len=2.0, n_near=16, n_far=20):
    """Piecewise Chebyshev-Lobatto nodes in rho: [0,h],[h,2h],[2h,4h], ... doubling up to seg_len
    (h = the smallest length scale of the radial functions), then segments of <= seg_len m up to
    rho_max.  Returns (nodes, segments) with segments [(a, b, node_idx)]."""
    edges = [0.0, h]
    while edges[-1] * 2 <= seg_len * (1 + 1e-12):
        edges.append(edges[-1] * 2)
    n_geo = len(edges) - 1
    while edges[-1] < rho_max:
        edges.append(min(rho_max, edges[-1] + seg_len) if rho_max - edges[-1] > 0.25 * seg_len
                     else rho_max)
        if edges[-1] >= rho_max:
            break
    edges = [e for e in edges if e <= max(rho_max, h)] if rho_max > 0 else [0.0, h]
    if edges[-1] < rho_max:
        edges.append(rho_max)
    nodes, segs = [], []
    for i, (a, b) in enumerate(zip(edges[:-1], edges[1:])):
        nn = n_near if i < n_geo else n_far
        t = np.cos(np.pi * np.arange(nn) / (nn - 1))[::-1]  # -1 .. 1
        x = 0.5 * (a + b) + 0.5 * (b - a) * t
        idx = np.arange(len(nodes), len(nodes) + nn)
        nodes.extend(x.tolist())
        segs.append((a, b, idx))
    return np.array(nodes), segs


def interp_matrix(segs, nodes, rho):
    """Barycentric Chebyshev-Lobatto interpolation matrix (len(rho), len(nodes))."""
    rho = np.asarray(rho, np.float64)
    Lm = np.zeros((len(rho), len(nodes)))
    for si, (a, b, idx) in enumerate(segs):
        last = si == len(segs) - 1
        sel = (rho >= a) & ((rho < b) | (last & (rho <= b + 1e-12 * max(1.0, b))))
        if not np.any(sel):
            continue
        x = nodes[idx]
        nn = len(idx)
        wb = (-1.0) ** np.arange(nn)
        wb[0] *= 0.5
        wb[-1] *= 0.5
        r = rho[sel]
        diff = r[:, None] - x[None, :]
        exact = diff == 0
        with np.errstate(divide="ignore", invalid="ignore"):
            q = wb[None, :] / diff
            q = q / q.sum(axis=1, keepdims=True)
        rows = np.where(exact.any(axis=1))[0]
        q[rows] = exact[rows].astype(np.float64)
        Lm[np.ix_(np.where(sel)[0], idx)] = q
    return Lm


def _bessel(ks, rho):
    """J0, J1, J2 of k rho for k (Q,) and rho (R,): each (Q, R)."""
    x = ks[:, None] * np.asarray(rho, np.float64)[None, :]
    return special.j0(x), special.j1(x), special.jv(2, x)


# --------------------------------------------------------------- homogeneous closed forms

def _green_E_hom(Rv, k, sigma):
    """Eq. 5 closed form (homogeneous, sigma) at nonzero offsets Rv (..., 3) -> (..., 3, 3)."""
    R = np.sqrt(np.sum(Rv * Rv, axis=-1))
    g = np.exp(1j * k * R) / (4 * np.pi * R)
    a = (k * k + 1j * k / R - 1.0 / R ** 2) * g / sigma
    b = (3.0 / R ** 2 - 3j * k / R - k * k) * g / sigma
    Rh = Rv / R[..., None]
    return a[..., None, None] * np.eye(3) + b[..., None, None] * (Rh[..., :, None] * Rh[..., None, :])


def _self_ball(k, sigma, dv):
    a = (3.0 * dv / (4.0 * np.pi)) ** (1.0 / 3.0)
    ika = 1j * k * a
    return ((2.0 / 3.0) * (1.0 - ika) * np.exp(ika) - 1.0) / sigma


def _E_mag_hom(Rv, m, k, omega):
    R = np.sqrt(np.sum(Rv * Rv, axis=-1))
    g = np.exp(1j * k * R) / (4 * np.pi * R)
    Rh = Rv / R[..., None]
    coef = 1j * omega * MU0 * g * (1j * k - 1.0 / R)
    return coef[..., None] * np.cross(Rh, np.broadcast_to(m, Rh.shape))


def _H_mag_hom(Rv, m, k):
    R = np.sqrt(np.sum(Rv * Rv, axis=-1))
    g = np.exp(1j * k * R) / (4 * np.pi * R)
    Rh = Rv / R[..., None]
    mm = np.broadcast_to(m, Rh.shape)
    a = (k * k + 1j * k / R - 1.0 / R ** 2) * g
    b = (3.0 / R ** 2 - 3j * k / R - k * k) * g
    return a[..., None] * mm + b[..., None] * Rh * np.sum(Rh * mm, axis=-1)[..., None]


# ------------------------------------------------------ electric dyadic: radial functions

_FUN = ("P0", "P2", "Q1", "R1", "Z0")


def _dyadic_coefs(med, sp_pair, n, m, k, un, um):
    """Per kind combo (kz, kzp): the five k-space integrand coefficients (without Bessel
    weights) of P0, P2, Q1, R1, Z0 for observer layer n, source layer m."""
    terms = sp_pair
    ss = med.sigma[n] * med.sigma[m]
    out = {}
    sgn = {"T": 1.0, "B": -1.0}
    for c, a, b in terms["TM"]:
        A = c * sgn[a] * un * sgn[b] * um / ss
        Bc = c * sgn[a] * un / ss
        Cc = c * sgn[b] * um / ss
        D = c / ss
        o = out.setdefault((a, b), [0j] * 5)
        o[0] = o[0] + A * k / (4 * np.pi)
        o[1] = o[1] + A * k / (4 * np.pi)
        o[2] = o[2] + Bc * k ** 2 / (2 * np.pi)
        o[3] = o[3] + Cc * k ** 2 / (2 * np.pi)
        o[4] = o[4] + D * k ** 3 / (2 * np.pi)
    for c, a, b in terms["TE"]:
        T = 1j * med.omega * MU0 * c
        o = out.setdefault((a, b), [0j] * 5)
        o[0] = o[0] + T * k / (4 * np.pi)
        o[1] = o[1] - T * k / (4 * np.pi)
    return out


def _blocks(alpha, edges=(0.0, 0.5, 1.0, 2.0, 4.0, np.inf)):
    """Index blocks of z by distance alpha to the relevant interface."""
    out = []
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = np.where((alpha >= lo) & (alpha < hi))[0]
        if len(sel):
            out.append((sel, float(alpha[sel].min())))
    return out


def dyadic_radial(med, z_obs, z_src, rho, h_min, order=_GL_ORDER):
    """Radial functions F[f][r, i, j] (f in P0,P2,Q1,R1,Z0) of the SECONDARY (same layer) or
    full (different layers) electric dyadic for observer depths z_obs[i], source depths z_src[j]
    and radial distances rho[r].  h_min: lower bound of the interface distances (zeta)."""
    z_obs = np.asarray(z_obs, np.float64)
    z_src = np.asarray(z_src, np.float64)
    rho = np.asarray(rho, np.float64)
    F = np.zeros((5, len(rho), len(z_obs), len(z_src)), np.complex128)
    lo = med.layer_of(z_obs)
    ls = med.layer_of(z_src)
    rmax = max(float(rho.max()), 1e-3)
    kmax_all = _ZETA_CUT / h_min
    width = min(np.pi / rmax, 4.0 / h_min)
    zmax = float(np.ptp(np.concatenate([z_obs, z_src]))) + 2 * h_min + 1.0
    k, wk = gl_nodes(kmax_all, width, order, zeta_max=zmax, kim_min=_kim(med))
    sp = (Spectral1D(med, k), Spectral1D(med.flipped(), k))
    J0, J1, J2 = _bessel(k, rho)
    Wb = [J0 * wk[:, None], J2 * wk[:, None], J1 * wk[:, None], J1 * wk[:, None], J0 * wk[:, None]]
    for n in np.unique(lo):
        io = np.where(lo == n)[0]
        for m in np.unique(ls):
            js = np.where(ls == m)[0]
            terms = _pair_terms(med, k, n, m, cache=sp)
            un, um = sp[0].u[:, n], sp[0].u[:, m]
            coefs = _dyadic_coefs(med, terms, n, m, k, un, um)
            for (a, b), cf in coefs.items():
                al = _alpha(med, n, a, z_obs[io])
                be = _alpha(med, m, b, z_src[js])
                extra = 0.0
                if n != m:  # the transmitted path crosses the intermediate layers
                    for j in range(min(n, m) + 1, max(n, m)):
                        extra += med.zt(j) - med.zb(j)
                for bi, amin in _blocks(al):
                    for bj, bmin in _blocks(be):
                        zeta = max(amin + bmin + extra, h_min)
                        q = int(np.searchsorted(k, _ZETA_CUT / zeta, side="right"))
                        if q == 0:
                            continue
                        Xo = _factor(med, un[:q], n, a, z_obs[io][bi])
                        Xs = _factor(med, um[:q], m, b, z_src[js][bj])
                        P = (Xo[:, :, None] * Xs[:, None, :]).reshape(q, -1)
                        for f in range(5):
                            V = Wb[f][:q] * cf[f][:q, None]  # (q, R)
                            F[f][np.ix_(np.arange(len(rho)), io[bi], js[bj])] += (V.T @ P).reshape(
                                len(rho), len(bi), len(bj))
    return F


def dyadic_at(med, r_obs, r_src, h_min=None, order=_GL_ORDER):
    """Full layered G^E (3x3) at individual point pairs (direct quadrature; test/reference
    use).  Primary closed form added for same-layer pairs.  r_obs, r_src: (P, 3)."""
    r_obs = np.atleast_2d(np.asarray(r_obs, np.float64))
    r_src = np.atleast_2d(np.asarray(r_src, np.float64))
    out = np.zeros((len(r_obs), 3, 3), np.complex128)
    for i, (ro, rs) in enumerate(zip(r_obs, r_src)):
        dx, dy = ro[0] - rs[0], ro[1] - rs[1]
        rho = np.hypot(dx, dy)
        n, m = med.layer_of(ro[2]), med.layer_of(rs[2])
        hm = h_min
        if hm is None:
            d = [abs(ro[2] - z) for z in med.zi] + [abs(rs[2] - z) for z in med.zi]
            hm = max(min(d) if d else 1.0, 1e-3)
        F = dyadic_radial(med, [ro[2]], [rs[2]], [rho], hm, order)[:, 0, 0, 0]
        out[i] = assemble_dyadic(F[:, None], np.array([dx]), np.array([dy]))[0]
        if n == m:
            out[i] += _green_E_hom(ro - rs, med.wavenumber(n), med.sigma[n])
    return out


def assemble_dyadic(F, dx, dy):
    """(..., 3, 3) tensors from the five radial functions F[f][...] at offsets (dx, dy)."""
    rho = np.hypot(dx, dy)
    with np.errstate(invalid="ignore", divide="ignore"):
        c = np.where(rho > 0, dx / np.where(rho > 0, rho, 1), 0.0)
        s = np.where(rho > 0, dy / np.where(rho > 0, rho, 1), 0.0)
    c2, s2 = c * c - s * s, 2 * s * c
    P0, P2, Q1, R1, Z0 = F
    shape = np.broadcast(P0, c).shape
    G = np.zeros(shape + (3, 3), np.complex128)
    G[..., 0, 0] = P0 - P2 * c2
    G[..., 1, 1] = P0 + P2 * c2
    G[..., 0, 1] = G[..., 1, 0] = -P2 * s2
    G[..., 0, 2] = -Q1 * c
    G[..., 1, 2] = -Q1 * s
    G[..., 2, 0] = R1 * c
    G[..., 2, 1] = R1 * s
    G[..., 2, 2] = Z0
    return G


# ----------------------------------------------------------------------------- the table

def layered_table(med, n, h, origin):
    """Quadrant table T[p, q, k, k', dj, di] (complex128, (3,3,nz,nz,ny,nx)) of the layered
    kernel samples: G^E_layered(r_k + (di dx, dj dy, 0), r_k') dv at cell centroids, the
    same-layer primary part the homogeneous Eq. 5 kernel of that layer with the equivolume
    ball self term (reading R3); the storage and mirror rules of reading R18."""
    nx, ny, nz = n
    dx, dy, dz = h
    dv = dx * dy * dz
    z = origin[2] + dz * np.arange(nz)
    lz = med.layer_of(z)
    dist = np.min(np.abs(z[:, None] - med.zi[None, :]), axis=1) if med.L > 1 else np.full(nz, np.inf)
    assert np.all(dist > 1e-9), "a cell centroid lies on an interface"
    T = np.zeros((3, 3, nz, nz, ny, nx), np.complex128)
    DI, DJ = np.meshgrid(np.arange(nx) * dx, np.arange(ny) * dy, indexing="xy")  # (ny, nx)
    # primary: same-layer pairs, homogeneous Eq. 5 of that layer (one evaluation per layer and
    # z offset, copied to every (k, k') pair with that offset)
    for j in np.unique(lz):
        kj = med.wavenumber(j)
        ks = np.where(lz == j)[0]
        for dk in range(-(len(ks) - 1), len(ks)):
            Rv = np.stack([DI, DJ, np.full_like(DI, dk * dz)], axis=-1)
            zero = (DI == 0) & (DJ == 0) & (dk == 0)
            Rv = np.where(zero[..., None], 1.0, Rv)
            G = _green_E_hom(Rv, kj, med.sigma[j]) * dv
            if zero.any():
                G[zero] = _self_ball(kj, med.sigma[j], dv) * np.eye(3)
            G = np.moveaxis(G, (-2, -1), (0, 1))
            for k in ks:
                kp = k - dk
                if kp in ks:
                    T[:, :, k, kp] = G
    if med.L == 1:
        return T
    # secondary (same layer) and transmitted (different layers) parts: radial functions on
    # Chebyshev nodes, interpolated to the lattice offsets
    rho_lat = np.hypot(DI, DJ)
    uniq, inv = np.unique(np.round(rho_lat / min(dx, dy), 9), return_inverse=True)
    rho_u = uniq * min(dx, dy)
    nodes, segs = radial_nodes(float(rho_u.max()), min(dx, dy))
    h_min = 2 * float(dist.min())
    F = dyadic_radial(med, z, z, nodes, h_min)  # (5, R, nz, nz)
    Lm = interp_matrix(segs, nodes, rho_u)  # (U, R)
    c = np.where(rho_lat > 0, DI / np.where(rho_lat > 0, rho_lat, 1), 0.0)
    s = np.where(rho_lat > 0, DJ / np.where(rho_lat > 0, rho_lat, 1), 0.0)
    c2, s2 = c * c - s * s, 2 * s * c
    inv = inv.reshape(ny, nx)
    R = len(nodes)
    for k in range(nz):
        Fk = F[:, :, k, :].transpose(1, 0, 2).reshape(R, -1)  # (R, 5 nz)
        Fk = (Lm @ Fk.real + 1j * (Lm @ Fk.imag)).reshape(-1, 5, nz).transpose(1, 0, 2)  # (5, U, nz)
        P0, P2, Q1, R1, Z0 = (Fk[f][inv] * dv for f in range(5))  # (ny, nx, nz)
        P0, P2, Q1, R1, Z0 = (np.moveaxis(a, -1, 0) for a in (P0, P2, Q1, R1, Z0))  # (nz', ny, nx)
        T[0, 0, k] += P0 - P2 * c2
        T[1, 1, k] += P0 + P2 * c2
        T[0, 1, k] += -P2 * s2
        T[1, 0, k] += -P2 * s2
        T[0, 2, k] += -Q1 * c
        T[1, 2, k] += -Q1 * s
        T[2, 0, k] += R1 * c
        T[2, 1, k] += R1 * s
        T[2, 2, k] += Z0
    return T


# ------------------------------------------------------------ magnetic-dipole background

def _mag_coefs(med, terms, n, m, k, un, um):
    """Per kind combo: E-field integrands (a = d_z G_TM/s_n, b = d_zs G_TE, c = G_TE,
    e = G_TM/s_n) for observer layer n, source layer m."""
    sgn = {"T": 1.0, "B": -1.0}
    out = {}
    for c, a, b in terms["TM"]:
        o = out.setdefault((a, b), [0j] * 4)
        o[0] = o[0] + c * sgn[a] * un / med.sigma[n]
        o[3] = o[3] + c / med.sigma[n]
    for c, a, b in terms["TE"]:
        o = out.setdefault((a, b), [0j] * 4)
        o[1] = o[1] + c * sgn[b] * um
        o[2] = o[2] + c
    return out


def incident_E_layered(med, points, src, moments, rho_interp=True):
    """E0 (complex, (n_mom, P, 3)) of magnetic dipoles with moments (n_mom, 3) at src in the
    layered medium, at points (P, 3).  Same-layer primary part closed form (reading R4)."""
    pts = np.atleast_2d(np.asarray(points, np.float64))
    src = np.asarray(src, np.float64)
    moments = np.atleast_2d(np.asarray(moments, np.float64))
    m = int(med.layer_of(src[2]))
    out = np.zeros((len(moments), len(pts), 3), np.complex128)
    zs = src[2]
    dxy = pts[:, :2] - src[None, :2]
    rho = np.hypot(dxy[:, 0], dxy[:, 1])
    zu, zinv = np.unique(pts[:, 2], return_inverse=True)
    lo = med.layer_of(zu)
    # radial functions at (rho nodes, z)
    dzi = np.abs(np.concatenate([zu[:, None] - med.zi[None, :]], axis=1)).min() if med.L > 1 else 1.0
    dsi = np.abs(zs - med.zi).min() if med.L > 1 else 1.0
    h_min = max(float(dzi) + float(dsi), 1e-4)
    if rho_interp:
        hseg = max(min(0.25, float(np.min(np.diff(zu))) if len(zu) > 1 else 0.25), 1e-3)
        nodes, segs = radial_nodes(max(float(rho.max()), hseg), hseg)
    else:
        nodes, segs = rho, None
    F = _mag_radial(med, zu, zs, nodes, h_min, m)  # (6, R, Z)
    if segs is not None:
        Lm = interp_matrix(segs, nodes, rho)
        Fp = np.einsum("pr,frz->fpz", Lm, F)  # (6, P, Z)
        Fp = Fp[:, np.arange(len(pts)), zinv]  # (6, P)
    else:
        Fp = F[:, np.arange(len(pts)), zinv]
    c = np.where(rho > 0, dxy[:, 0] / np.where(rho > 0, rho, 1), 0.0)
    s = np.where(rho > 0, dxy[:, 1] / np.where(rho > 0, rho, 1), 0.0)
    c2, s2 = c * c - s * s, 2 * s * c
    F0a, F2a, F0b, F2b, F1c, F1e = Fp
    iwm = 1j * med.omega * MU0
    for t, mm in enumerate(moments):
        mx, my, mz = mm
        Ex = mx * (-F2a * s2 - F2b * s2) + my * (-F0a + F2a * c2 + F0b + F2b * c2) + mz * (-F1c * s)
        Ey = mx * (F0a + F2a * c2 - F0b + F2b * c2) + my * (F2a * s2 + F2b * s2) + mz * (F1c * c)
        Ez = mx * (F1e * s) - my * (F1e * c)
        out[t] = iwm * np.stack([Ex, Ey, Ez], axis=-1)
        same = lo[zinv] == m
        if same.any():
            out[t][same] += _E_mag_hom(pts[same] - src, mm, med.wavenumber(m), med.omega)
    return out


def incident_E_layered_grid(med, x, y, z, src, moments):
    """E0 on a tensor grid of cell centroids: (n_mom, 3, nz, ny, nx) complex128 -- the radial
    functions are computed once per depth and interpolated to the (x, y) columns."""
    x, y, z = (np.asarray(a, np.float64) for a in (x, y, z))
    src = np.asarray(src, np.float64)
    moments = np.atleast_2d(np.asarray(moments, np.float64))
    m = int(med.layer_of(src[2]))
    nx, ny, nz = len(x), len(y), len(z)
    DX, DY = np.meshgrid(x - src[0], y - src[1], indexing="xy")  # (ny, nx)
    rho = np.hypot(DX, DY).ravel()
    lo = med.layer_of(z)
    if med.L > 1:
        dz = np.abs(z[:, None] - med.zi[None, :]).min()
        ds = np.abs(src[2] - med.zi).min()
        h_min = max(float(dz) + float(ds), 1e-4)
    else:
        h_min = 1.0
    # radial segments start at the smallest length scale: the cell size or the source-to-interface
    # plus cell-to-interface distance (a source next to an interface)
    hseg = min(abs(x[1] - x[0]) if nx > 1 else 0.25, abs(y[1] - y[0]) if ny > 1 else 0.25, h_min)
    out = np.zeros((len(moments), 3, nz, ny, nx), np.complex128)
    iwm = 1j * med.omega * MU0
    if med.L > 1 or m != 0:
        nodes, segs = radial_nodes(max(float(rho.max()), hseg), hseg)
        F = _mag_radial(med, z, src[2], nodes, h_min, m)  # (6, R, nz)
        Lm = interp_matrix(segs, nodes, rho)  # (ny nx, R)
        R = len(nodes)
        Fr = F.transpose(1, 0, 2).reshape(R, -1)
        Fp = (Lm @ Fr.real + 1j * (Lm @ Fr.imag)).reshape(ny, nx, 6, nz).transpose(2, 3, 0, 1)  # (6, nz, ny, nx)
        c = np.where(rho > 0, DX.ravel() / np.where(rho > 0, rho, 1), 0.0).reshape(ny, nx)
        s_ = np.where(rho > 0, DY.ravel() / np.where(rho > 0, rho, 1), 0.0).reshape(ny, nx)
        c2, s2 = c * c - s_ * s_, 2 * s_ * c
        F0a, F2a, F0b, F2b, F1c, F1e = Fp
        for t, mm in enumerate(moments):
            mx, my, mz = mm
            out[t, 0] = iwm * (mx * (-F2a * s2 - F2b * s2) + my * (-F0a + F2a * c2 + F0b + F2b * c2) + mz * (-F1c * s_))
            out[t, 1] = iwm * (mx * (F0a + F2a * c2 - F0b + F2b * c2) + my * (F2a * s2 + F2b * s2) + mz * (F1c * c))
            out[t, 2] = iwm * (mx * (F1e * s_) - my * (F1e * c))
    ks = np.where(lo == m)[0]
    if len(ks):
        Z, Y, X = np.meshgrid(z[ks], y, x, indexing="ij")
        Rv = np.stack([X, Y, Z], axis=-1) - src
        for t, mm in enumerate(moments):
            out[t][:, ks] += np.moveaxis(_E_mag_hom(Rv, mm, med.wavenumber(m), med.omega), -1, 0)
    return out


def _mag_radial(med, zu, zs, rho, h_min, m, order=_GL_ORDER):
    """F (6, R, Z): F0(a), F2(a), F0(b), F2(b), F1(c), F1(e) for observer depths zu."""
    rmax = max(float(np.max(rho)), 1e-3)
    kmax_all = _ZETA_CUT / h_min
    width = min(np.pi / rmax, 4.0 / h_min)
    zmax = float(np.ptp(np.append(zu, zs))) + 2 * h_min + 1.0
    k, wk = gl_nodes(kmax_all, width, order, zeta_max=zmax, kim_min=_kim(med))
    sp = (Spectral1D(med, k), Spectral1D(med.flipped(), k))
    J0, J1, J2 = _bessel(k, rho)
    lo = med.layer_of(zu)
    F = np.zeros((6, len(rho), len(zu)), np.complex128)
    for n in np.unique(lo):
        io = np.where(lo == n)[0]
        terms = _pair_terms(med, k, n, m, cache=sp)
        un, um = sp[0].u[:, n], sp[0].u[:, m]
        coefs = _mag_coefs(med, terms, n, m, k, un, um)
        extra = 0.0
        for j in range(min(n, m) + 1, max(n, m)):
            extra += med.zt(j) - med.zb(j)
        for (a, b), cf in coefs.items():
            al = _alpha(med, n, a, zu[io])
            be = float(_alpha(med, m, b, np.array([zs]))[0])
            for bi, amin in _blocks(al):
                zeta = max(amin + be + extra, h_min)
                q = int(np.searchsorted(k, _ZETA_CUT / zeta, side="right"))
                if q == 0:
                    continue
                Xo = _factor(med, un[:q], n, a, zu[io][bi])
                Xs = _factor(med, um[:q], m, b, np.array([zs]))
                X = Xo * Xs  # (q, nb)
                w1 = (wk * k / (4 * np.pi))[:q, None]
                w2 = (wk * k ** 2 / (2 * np.pi))[:q, None]
                sel = np.ix_(np.arange(len(rho)), io[bi])
                F[0][sel] += ((J0[:q] * w1 * cf[0][:q, None]).T @ X)
                F[1][sel] += ((J2[:q] * w1 * cf[0][:q, None]).T @ X)
                F[2][sel] += ((J0[:q] * w1 * cf[1][:q, None]).T @ X)
                F[3][sel] += ((J2[:q] * w1 * cf[1][:q, None]).T @ X)
                F[4][sel] += ((J1[:q] * w2 * cf[2][:q, None]).T @ X)
                F[5][sel] += ((J1[:q] * w2 * cf[3][:q, None]).T @ X)
    return F


def incident_H_layered(med, points, src, moments, order=_GL_ORDER):
    """H0 (complex, (n_mom, P, 3)) of magnetic dipoles at src in the layered medium at a few
    points (direct quadrature per point)."""
    pts = np.atleast_2d(np.asarray(points, np.float64))
    src = np.asarray(src, np.float64)
    moments = np.atleast_2d(np.asarray(moments, np.float64))
    m = int(med.layer_of(src[2]))
    out = np.zeros((len(moments), len(pts), 3), np.complex128)
    sgn = {"T": 1.0, "B": -1.0}
    iwm = 1j * med.omega * MU0
    for p, r in enumerate(pts):
        n = int(med.layer_of(r[2]))
        dx, dy = r[0] - src[0], r[1] - src[1]
        rho = np.hypot(dx, dy)
        d = [abs(r[2] - z) + abs(src[2] - z) for z in med.zi]
        hm = max(min(d) if d else 1.0, 1e-4)
        zmax = abs(r[2] - src[2]) + 2 * hm + 1.0
        k, wk = gl_nodes(_ZETA_CUT / hm, min(np.pi / max(rho, 1e-3), 4.0 / hm), order, zeta_max=zmax, kim_min=_kim(med))
        sp = (Spectral1D(med, k), Spectral1D(med.flipped(), k))
        terms = _pair_terms(med, k, n, m, cache=sp)
        un, um = sp[0].u[:, n], sp[0].u[:, m]
        # alpha = d_z d_zs G_TE, beta = d_z G_TE, gamma = d_zs G_TE, dlt = G_TE, eps = i w mu0 G_TM
        acc = {key: np.zeros_like(k, dtype=np.complex128) for key in ("al", "be", "ga", "dl", "ep")}
        for c, a, b in terms["TE"]:
            Xo = _factor(med, un, n, a, np.array([r[2]]))
            Xs = _factor(med, um, m, b, np.array([src[2]]))
            X = (Xo * Xs)[:, 0]
            acc["al"] += c * sgn[a] * un * sgn[b] * um * X
            acc["be"] += c * sgn[a] * un * X
            acc["ga"] += c * sgn[b] * um * X
            acc["dl"] += c * X
        for c, a, b in terms["TM"]:
            Xo = _factor(med, un, n, a, np.array([r[2]]))
            Xs = _factor(med, um, m, b, np.array([src[2]]))
            acc["ep"] += iwm * c * (Xo * Xs)[:, 0]
        x = k * rho
        J0, J1, J2 = special.j0(x), special.j1(x), special.jv(2, x)

        def F0(f):
            return np.sum(wk * f * J0 * k) / (4 * np.pi)

        def F2(f):
            return np.sum(wk * f * J2 * k) / (4 * np.pi)

        def F1(f):
            return np.sum(wk * f * J1 * k ** 2) / (2 * np.pi)

        def F0p(f):
            return np.sum(wk * f * J0 * k ** 3) / (2 * np.pi)

        c_, s_ = (dx / rho, dy / rho) if rho > 0 else (0.0, 0.0)
        c2, s2 = c_ * c_ - s_ * s_, 2 * s_ * c_
        al, be, ga, dl, ep = (acc[key] for key in ("al", "be", "ga", "dl", "ep"))
        F0al, F2al, F0ep, F2ep = F0(al), F2(al), F0(ep), F2(ep)
        F1be, F1ga, F0pdl = F1(be), F1(ga), F0p(dl)
        for t, mm in enumerate(moments):
            mx, my, mz = mm
            Hx = mx * (F0al - F2al * c2 + F0ep + F2ep * c2) + my * (-F2al * s2 + F2ep * s2) + mz * (-F1be * c_)
            Hy = mx * (-F2al * s2 + F2ep * s2) + my * (F0al + F2al * c2 + F0ep - F2ep * c2) + mz * (-F1be * s_)
            Hz = mx * (F1ga * c_) + my * (F1ga * s_) + mz * F0pdl
            out[t, p] = (Hx, Hy, Hz)
            if n == m:
                out[t, p] += _H_mag_hom(r - src, mm, med.wavenumber(m))
    return out
