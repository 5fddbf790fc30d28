"""Contraction-IE right preconditioner (oracle; test infrastructure only).

SURVEY 8(f)-2, the remedy the paper cites for high contrast: with the per-cell
change of unknown chi = a E, a = (sigma + sigma_b I) / (2 sigma_b) (Hursan & Zhdanov's
contraction integral equation), Eq. 8 becomes (I - G dsigma) P chi = E0 with P = a^-1 =
2 sigma_b (sigma + sigma_b I)^-1: the same solution E = P chi and the same Eq. 9 residual.
"""

import numpy as np


def contraction_P(sigma, sigma_b):
    """P = 2 sigma_b (sigma + sigma_b I)^-1 per cell; sigma (..., 3, 3), sigma_b scalar or (...)"""
    sb = np.asarray(sigma_b, np.float64)[..., None, None] if np.ndim(sigma_b) else float(sigma_b)
    return 2.0 * sb * np.linalg.inv(np.asarray(sigma, np.float64) + sb * np.eye(3))


def apply_cellwise(M, E):
    """(M E) per cell: M (nz, ny, nx, 3, 3), E (3, nz, ny, nx)."""
    return np.einsum("zyxpq,qzyx->pzyx", M, E)
