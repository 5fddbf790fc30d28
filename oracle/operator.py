"""The discrete IE operator (I - G dsigma) of Eq. 8 (oracle; test infrastructure only).

Three independent evaluations, each written plainly:
  * ``dense_matrix``  -- the 3N x 3N matrix of Eq. 8 assembled entry by entry from the
                         kernel samples; tiny grids only.
  * ``direct_rows``   -- Eq. 3 discretised as a literal sum over cells, for selected
                         output cells (any grid size; O(N) per output cell).
  * ``fft_apply``     -- Eq. 10: G_pq J_q = F^-1( F[G_pq] . F[J_q] ) with 2x zero padding
                         per axis, numpy FFTs of the full padded grid.

Field layout (3, nz, ny, nx); dsigma layout (nz, ny, nx, 3, 3).
"""

import numpy as np
import scipy.fft as sfft

from ._threads import WORKERS

from . import physics


def contrast_source(dsigma, E):
    """J = dsigma E per cell (the contrast source of Eq. 3).  E: (3,nz,ny,nx)."""
    return np.einsum("zyxpq,qzyx->pzyx", dsigma, E)


def dense_matrix(n, h, k0, sigma_b, dsigma):
    """A = I - K D  (Eq. 8), rows/cols ordered (component, z, y, x)."""
    nx, ny, nz = n
    N = nx * ny * nz
    K = physics.kernel_offsets(n, h, k0, sigma_b)  # (2nz-1, 2ny-1, 2nx-1, 3, 3)
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    iz, iy, ix = iz.ravel(), iy.ravel(), ix.ravel()
    dz = iz[:, None] - iz[None, :] + nz - 1
    dy = iy[:, None] - iy[None, :] + ny - 1
    dx = ix[:, None] - ix[None, :] + nx - 1
    Kcc = K[dz, dy, dx]  # (N, N, 3, 3): K(r_c - r_c')
    Kmat = Kcc.transpose(2, 0, 3, 1).reshape(3 * N, 3 * N)
    D = np.zeros((3 * N, 3 * N))
    ds = dsigma.reshape(N, 3, 3)
    for p in range(3):
        for q in range(3):
            D[p * N + np.arange(N), q * N + np.arange(N)] = ds[:, p, q]
    return np.eye(3 * N) - Kmat @ D


def direct_rows(n, h, k0, sigma_b, dsigma, E, cells, identity=True):
    """(I - G dsigma) E evaluated at output cells ``cells`` = list of (ix, iy, iz) by direct
    summation over every source cell (Eq. 3 discretised).  Returns (len(cells), 3)."""
    nx, ny, nz = n
    dv = h[0] * h[1] * h[2]
    J = contrast_source(dsigma, E)  # (3, nz, ny, nx)
    out = np.zeros((len(cells), 3), np.complex128)
    slab = max(1, (1 << 20) // (nx * ny))  # sum over z-slabs to bound memory on large grids
    for t, (cx, cy, cz) in enumerate(cells):
        s = np.zeros(3, np.complex128)
        for z0 in range(0, nz, slab):
            z1 = min(nz, z0 + slab)
            iz, iy, ix = np.meshgrid(np.arange(z0, z1), np.arange(ny), np.arange(nx), indexing="ij")
            Rv = np.stack([(cx - ix) * h[0], (cy - iy) * h[1], (cz - iz) * h[2]], axis=-1)
            zero = (ix == cx) & (iy == cy) & (iz == cz)
            Rv_safe = np.where(zero[..., None], 1.0, Rv)
            K = physics.green_E(Rv_safe, k0, sigma_b) * dv
            K[zero] = physics.self_term(k0, sigma_b, dv)
            s += np.einsum("zyxpq,qzyx->p", K, J[:, z0:z1])
        out[t] = (E[:, cz, cy, cx] if identity else 0.0) - s
    return out


def green_spectra(n, h, k0, sigma_b):
    """F[G_pq] on the 2x padded grid (Eq. 10): the kernel samples are placed in a
    circulant embedding of size (2nz, 2ny, 2nx) -- offset d at index d mod 2n, the unused
    slot at offset n set to 0 (reading R5) -- then fftn.  Returns (3, 3, 2nz, 2ny, 2nx)."""
    nx, ny, nz = n
    K = physics.kernel_offsets(n, h, k0, sigma_b)
    C = np.zeros((3, 3, 2 * nz, 2 * ny, 2 * nx), np.complex128)
    dz = np.arange(-(nz - 1), nz) % (2 * nz)
    dy = np.arange(-(ny - 1), ny) % (2 * ny)
    dx = np.arange(-(nx - 1), nx) % (2 * nx)
    C[:, :, dz[:, None, None], dy[None, :, None], dx[None, None, :]] = K.transpose(3, 4, 0, 1, 2)
    return sfft.fftn(C, axes=(2, 3, 4), workers=WORKERS)


def fft_scatter(Ghat, dsigma, E, n):
    """G (dsigma E) on the grid via Eq. 10: pad J to 2n, FFT, multiply by F[G_pq], sum over
    q, inverse FFT, crop to the original cells."""
    nx, ny, nz = n
    J = contrast_source(dsigma, E)
    Jp = np.zeros((3, 2 * nz, 2 * ny, 2 * nx), np.complex128)
    Jp[:, :nz, :ny, :nx] = J
    Jh = sfft.fftn(Jp, axes=(1, 2, 3), workers=WORKERS)
    Yh = np.einsum("pqzyx,qzyx->pzyx", Ghat, Jh)
    Y = sfft.ifftn(Yh, axes=(1, 2, 3), workers=WORKERS)
    return Y[:, :nz, :ny, :nx]


def fft_apply(Ghat, dsigma, E, n):
    """(I - G dsigma) E  (Eq. 8) with the convolution of Eq. 10."""
    return E - fft_scatter(Ghat, dsigma, E, n)


class Operator:
    """Matrix-free A = I - G dsigma on one rectangular domain (full grid or a box)."""

    def __init__(self, n, h, k0, sigma_b, dsigma):
        self.n = tuple(n)
        self.dsigma = dsigma
        self.Ghat = green_spectra(n, h, k0, sigma_b)

    def scatter(self, E):
        return fft_scatter(self.Ghat, self.dsigma, E, self.n)

    def __call__(self, E):
        return E - self.scatter(E)


def relative_residual(A, E, E0):
    """e = ||E0 - (I - G dsigma) E|| / ||E0||   (Eq. 9), L2 over all cells of the
    operator's domain (reading R7)."""
    return np.linalg.norm((E0 - A(E)).ravel()) / np.linalg.norm(E0.ravel())
