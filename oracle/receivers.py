"""Receiver magnetic fields, Eq. 4 with Eq. 6 (oracle; test infrastructure only).

H(r) = H^(0)(r) + sum_c G^H(r, r_c) dsigma_c E_c dv   (Eq. 4; "straightforward
addition").  With Eq. 6, G^H J = (i omega mu0)^-1 curl(G^E J) = grad g x J, so the
scattered part is sum_c g(R)(i k0 - 1/R) (Rhat x J_c) dv with R = r - r_c; a term with
R = 0 is 0 (odd kernel over the equivolume ball; reading R13).
Voltage of a unit receiver coil along m_r: V = i omega mu0 m_r . H (reading R14), pinned by
Faraday's law (Eq. 1) in tests/test_oracle_pins.py: it equals the loop integral of E around a
small coil of area |m_r|, sign included, for the incident and the scattered fields.
"""

import numpy as np

from . import physics
from .operator import contrast_source


def receiver_H(n, h, origin, k0, sigma_b, dsigma, E, rx, src_pos, moment):
    """H at receiver points rx (n_rx, 3) for one source dipole.  Returns (n_rx, 3) complex."""
    dv = h[0] * h[1] * h[2]
    J = contrast_source(dsigma, E)  # (3, nz, ny, nx)
    rc = physics.centroids(n, h, origin)  # (nz, ny, nx, 3)
    out = np.zeros((len(rx), 3), np.complex128)
    for t, r in enumerate(np.asarray(rx, np.float64)):
        Rv = r - rc
        R = np.sqrt(np.sum(Rv * Rv, axis=-1))
        zero = R == 0.0
        Rs = np.where(zero, 1.0, R)
        coef = physics.scalar_green(Rs, k0) * (1j * k0 - 1.0 / Rs) * dv
        coef = np.where(zero, 0.0, coef)
        Rh = Rv / Rs[..., None]
        Jc = np.moveaxis(J, 0, -1)
        sc = np.sum(coef[..., None] * np.cross(Rh, Jc), axis=(0, 1, 2))
        out[t] = physics.incident_H(r, src_pos, moment, k0) + sc
    return out


def voltage(H, m_r, freq_hz):
    """V = i omega mu0 m_r . H (EMF of a coil of area |m_r| along m_r; reading R14; pinned by the
    Faraday loop integral, tests/test_oracle_pins.py)."""
    return 1j * physics.omega_of(freq_hz) * physics.MU0 * np.sum(np.asarray(m_r) * H, axis=-1)
