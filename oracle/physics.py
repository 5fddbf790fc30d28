"""Closed-form physics of the homogeneous-background IE (oracle; test infrastructure only).

Citations are PAPER.md line numbers ("P:n") with the equation they fall in.

Conventions (Eq. 1-2): time dependence e^{-i omega t}, mu = mu0, the displacement
current is dropped (diffusive regime), background is homogeneous isotropic sigma_b.
"""

import numpy as np

# mu0 = 4 pi 1e-7 H/m exactly (reading R1; CODATA differs at 1e-10 relative).
MU0 = 4e-7 * np.pi


def omega_of(freq_hz):
    return 2.0 * np.pi * float(freq_hz)


def wavenumber(sigma_b, freq_hz):
    """k0 = sqrt(i omega mu0 sigma0)  (text after Eq. 7).

    Principal branch: Re k0 > 0 and Im k0 > 0, so e^{i k0 R} decays (reading R2).
    """
    k0 = np.sqrt(1j * omega_of(freq_hz) * MU0 * float(sigma_b))
    assert k0.real > 0 and k0.imag > 0
    return complex(k0)


def scalar_green(R, k0):
    """g(R) = e^{i k0 R} / (4 pi R)   (Eq. 7)."""
    R = np.asarray(R, dtype=np.float64)
    return np.exp(1j * k0 * R) / (4.0 * np.pi * R)


def green_E(Rvec, k0, sigma_b):
    """Electric Green's tensor G^E(R) = (i omega mu0 I + grad grad / sigma0) g   (Eq. 5).

    Written out with k0^2 = i omega mu0 sigma0 (so i omega mu0 = k0^2 / sigma0):
        sigma0 G^E = g [ (k0^2 + i k0/R - 1/R^2) I + (3/R^2 - 3 i k0/R - k0^2) Rhat Rhat^T ].
    ``Rvec``: (..., 3) nonzero offsets r - r'.  Returns (..., 3, 3) complex.
    """
    Rvec = np.asarray(Rvec, dtype=np.float64)
    R = np.sqrt(np.sum(Rvec * Rvec, axis=-1))
    g = scalar_green(R, k0)
    a = (k0 * k0 + 1j * k0 / R - 1.0 / R ** 2) * g / sigma_b
    b = (3.0 / R ** 2 - 3j * k0 / R - k0 * k0) * g / sigma_b
    Rh = Rvec / R[..., None]
    eye = np.eye(3)
    return a[..., None, None] * eye + b[..., None, None] * (Rh[..., :, None] * Rh[..., None, :])


def self_term(k0, sigma_b, dv):
    """Integral of G^E over the equivolume sphere of the singular cell.

    P:64 states the method (integrate the Green's function of a single grid block over a
    sphere of equal volume) but not the result; reading R3 in DESIGN.md:
        K(0) = (1/sigma_b) [ (2/3)(1 - i k0 a) e^{i k0 a} - 1 ] I,   a = (3 dv / 4 pi)^{1/3}.
    Pinned in tests against a 3-D spherical quadrature of Eq. 5 plus the textbook
    depolarisation term -I/(3 sigma_b) (static limit).
    """
    a = (3.0 * dv / (4.0 * np.pi)) ** (1.0 / 3.0)
    ika = 1j * k0 * a
    return ((2.0 / 3.0) * (1.0 - ika) * np.exp(ika) - 1.0) / sigma_b * np.eye(3)


def centroids(n, h, origin):
    """Cell centroids r^j.  n=(nx,ny,nz), h=(dx,dy,dz), origin = centroid of cell (0,0,0).
    Returns (nz, ny, nx, 3)."""
    nx, ny, nz = n
    x = origin[0] + h[0] * np.arange(nx)
    y = origin[1] + h[1] * np.arange(ny)
    z = origin[2] + h[2] * np.arange(nz)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return np.stack([X, Y, Z], axis=-1)


def kernel_offsets(n, h, k0, sigma_b):
    """Discrete kernel K(d) = G^E(d*h) * dv for every lattice offset d in (-n, n) per axis
    (midpoint rule off the diagonal; reading R3 for d = 0).

    Returns (2nz-1, 2ny-1, 2nx-1, 3, 3) complex, index [dz+nz-1, dy+ny-1, dx+nx-1].
    """
    nx, ny, nz = n
    dv = h[0] * h[1] * h[2]
    dz = np.arange(-(nz - 1), nz) * h[2]
    dy = np.arange(-(ny - 1), ny) * h[1]
    dx = np.arange(-(nx - 1), nx) * h[0]
    Z, Y, X = np.meshgrid(dz, dy, dx, indexing="ij")
    Rv = np.stack([X, Y, Z], axis=-1)
    zero = (X == 0) & (Y == 0) & (Z == 0)
    Rv_safe = np.where(zero[..., None], 1.0, Rv)
    K = green_E(Rv_safe, k0, sigma_b) * dv
    K[zero] = self_term(k0, sigma_b, dv)
    return K


def incident_E(points, src_pos, moment, k0, freq_hz):
    """Background E of a magnetic dipole m at r_s in the homogeneous full space:
    E0 = i omega mu0 grad g x m = i omega mu0 g (i k0 - 1/R) (Rhat x m),  R = r - r_s.

    The paper uses E^(0) (Eq. 3) without printing it (reading R4); pinned by curl
    consistency with ``incident_H`` (Eq. 1: curl E = i omega mu H) and the static limits.
    ``points``: (..., 3).  Returns (..., 3) complex.
    """
    Rv = np.asarray(points, np.float64) - np.asarray(src_pos, np.float64)
    R = np.sqrt(np.sum(Rv * Rv, axis=-1))
    g = scalar_green(R, k0)
    Rh = Rv / R[..., None]
    m = np.broadcast_to(np.asarray(moment, np.float64), Rh.shape)
    coef = 1j * omega_of(freq_hz) * MU0 * g * (1j * k0 - 1.0 / R)
    return coef[..., None] * np.cross(Rh, m)


def incident_H(points, src_pos, moment, k0):
    """Background H of the same dipole: H0 = (k0^2 + grad grad) g m = sigma0 G^E(R) m
    (from Eq. 1 with Eq. 5; reading R4).  Returns (..., 3) complex."""
    Rv = np.asarray(points, np.float64) - np.asarray(src_pos, np.float64)
    R = np.sqrt(np.sum(Rv * Rv, axis=-1))
    g = scalar_green(R, k0)
    Rh = Rv / R[..., None]
    m = np.broadcast_to(np.asarray(moment, np.float64), Rh.shape)
    a = (k0 * k0 + 1j * k0 / R - 1.0 / R ** 2) * g
    b = (3.0 / R ** 2 - 3j * k0 / R - k0 * k0) * g
    return a[..., None] * m + b[..., None] * Rh * np.sum(Rh * m, axis=-1)[..., None]


def contrast(sigma, sigma_b):
    """Delta sigma = sigma - sigma0 I.  sigma: (..., 3, 3)."""
    return np.asarray(sigma, np.float64) - float(sigma_b) * np.eye(3)
