"""Building blocks of the synthetic conductivity models (inputs only)."""

import numpy as np


def vti_tensor(sigma_h, sigma_v, theta, phi):
    """Rotated transversely-isotropic conductivity tensor, Appendix C:
        s'_xx = s_h + (s_v - s_h) sin^2(th) cos^2(ph)     s'_xy = (s_v - s_h) sin^2(th) sin(ph) cos(ph)
        s'_xz = (s_v - s_h) sin(th) cos(th) cos(ph)       s'_yy = s_h + (s_v - s_h) sin^2(th) sin^2(ph)
        s'_yz = (s_v - s_h) sin(th) cos(th) sin(ph)       s'_zz = s_v - (s_v - s_h) sin^2(th)
    theta = dip (tilt of the symmetry axis from z), phi = azimuth (reading R15: the
    formulas, not P:440's axis names, fix the meaning).  Broadcasts; returns (..., 3, 3).
    """
    sh, sv, th, ph = np.broadcast_arrays(*(np.asarray(v, np.float64) for v in (sigma_h, sigma_v, theta, phi)))
    d = sv - sh
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    out = np.empty(sh.shape + (3, 3))
    out[..., 0, 0] = sh + d * st ** 2 * cp ** 2
    out[..., 0, 1] = out[..., 1, 0] = d * st ** 2 * sp * cp
    out[..., 0, 2] = out[..., 2, 0] = d * st * ct * cp
    out[..., 1, 1] = sh + d * st ** 2 * sp ** 2
    out[..., 1, 2] = out[..., 2, 1] = d * st * ct * sp
    out[..., 2, 2] = sv - d * st ** 2
    return out


def haar_rotation(rng):
    """Random rotation, Haar-distributed: QR of a 3x3 N(0,1) matrix, column signs fixed by
    diag(R) > 0, det forced to +1 by flipping the last column."""
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(R))[None, :]
    if np.linalg.det(Q) < 0:
        Q[:, 2] = -Q[:, 2]
    return Q


def gaussian_random_field(rng, shape, h, corr_len):
    """N(0,1) white noise filtered by exp(-|k|^2 l^2 / 4) (covariance exp(-r^2 / 2 l^2)),
    then normalised to zero mean, unit std.  shape = (nz, ny, nx)."""
    w = rng.standard_normal(shape)
    kz = 2 * np.pi * np.fft.fftfreq(shape[0], h)
    ky = 2 * np.pi * np.fft.fftfreq(shape[1], h)
    kx = 2 * np.pi * np.fft.rfftfreq(shape[2], h)
    K2 = kz[:, None, None] ** 2 + ky[None, :, None] ** 2 + kx[None, None, :] ** 2
    f = np.fft.irfftn(np.fft.rfftn(w) * np.exp(-K2 * corr_len ** 2 / 4.0), s=shape, axes=(0, 1, 2))
    f -= f.mean()
    f /= f.std()
    return f


def tool_frame(incl_deg, azim_deg):
    """Tool axes for a straight trajectory: z' along the hole d = (sin i cos a, sin i sin a,
    cos i), x' = high side (cos i cos a, cos i sin a, -sin i), y' = z' x x'.  Rows x', y', z'."""
    i, a = np.radians(incl_deg), np.radians(azim_deg)
    zp = np.array([np.sin(i) * np.cos(a), np.sin(i) * np.sin(a), np.cos(i)])
    xp = np.array([np.cos(i) * np.cos(a), np.cos(i) * np.sin(a), -np.sin(i)])
    yp = np.cross(zp, xp)
    return np.stack([xp, yp, zp])


def box_grid(n, splits):
    """Equal rectangular partition (Eq. 11) of an (nx, ny, nz) grid into splits = (sx, sy, sz)
    boxes, x-fastest order.  Box = (i0, i1, j0, j1, k0, k1)."""
    nx, ny, nz = n
    sx, sy, sz = splits
    bx, by, bz = nx // sx, ny // sy, nz // sz
    assert bx * sx == nx and by * sy == ny and bz * sz == nz
    boxes = []
    for k in range(sz):
        for j in range(sy):
            for i in range(sx):
                boxes.append((i * bx, (i + 1) * bx, j * by, (j + 1) * by, k * bz, (k + 1) * bz))
    return boxes
