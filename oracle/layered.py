"""The IE operator over a horizontally layered background given as a host table of kernel
samples (oracle; test infrastructure only).

The paper's background is homogeneous; BASELINE.json c3/c4 ask for layered
backgrounds with "layered Green's-tensor tables ... precomputed on the host as input data
for both paths".  For a horizontally layered medium the discrete kernel is translation
invariant in x and y only, so Eq. 3 discretised reads (reading R17)

    (G J)_p(i,j,k) = sum_{q,i',j',k'} T_pq(i-i', j-j'; k, k') J_q(i',j',k'),
    dsigma = sigma - sigma_b(z_k) I

with T the table (kernel samples including dv and the self term, the layered analogue of
K(d) in operator.py).  Storage (reading R18): the quadrant of non-negative offsets,
complex128 [3][3][nz][nz][ny][nx] = T[p, q, k, k', dj, di]; negative offsets follow the
mirror symmetry of a horizontally layered isotropic medium,
    T_pq(-di, dj) = sx_p sx_q T_pq(di, dj),  sx = (-1, 1, 1),
    T_pq(di, -dj) = sy_p sy_q T_pq(di, dj),  sy = (1, -1, 1),
so components odd in x (xy, xz) vanish at di = 0 and those odd in y (xy, yz) at dj = 0 (the
stored values there are ignored).

Evaluations, written plainly:
  * ``dense_matrix_layered`` -- the 3N x 3N matrix entry by entry (tiny grids);
  * ``LayeredOperator``      -- 2x zero padding in x and y only, numpy fft2 of the
                                circulant-embedded table per (p, q, k, k'), a dense
                                (3nz x 3nz) contraction per horizontal wavenumber, ifft2.
Tables: ``homogeneous_table`` (the degenerate equal-layer table: every layer sigma_b,
T = K(di, dj, k - k') of operator.py; pins the machinery against Eq. 10) and
``random_table`` (arbitrary values, for brute-force checks).  A physical layered table
(Sommerfeld integrals of the 1-D layered medium) is not built: parity unpinned, R19.
"""

import numpy as np
import scipy.fft as sfft

from ._threads import WORKERS

from . import physics

SX = np.array([-1.0, 1.0, 1.0])
SY = np.array([1.0, -1.0, 1.0])


def expand_table(Tq):
    """Quadrant table (3,3,nz,nz,ny,nx) -> full offsets (3,3,nz,nz,2ny-1,2nx-1), index
    [.., dj + ny - 1, di + nx - 1], by the mirror rules (R18)."""
    _, _, nz, _, ny, nx = Tq.shape
    F = np.zeros((3, 3, nz, nz, 2 * ny - 1, 2 * nx - 1), np.complex128)
    sx = np.outer(SX, SX)[:, :, None, None, None, None]
    sy = np.outer(SY, SY)[:, :, None, None, None, None]
    # at zero offset the rules force the odd components to vanish (f(0) = -f(0)); the
    # stored values there are ignored
    Tq = Tq.copy()
    Tq[..., :, 0] *= (sx[..., 0, 0] > 0)[..., None]
    Tq[..., 0, :] *= (sy[..., 0, 0] > 0)[..., None]
    F[..., ny - 1:, nx - 1:] = Tq                                   # di >= 0, dj >= 0
    F[..., ny - 1:, :nx - 1] = sx * Tq[..., :, :0:-1]               # di < 0
    F[..., :ny - 1, nx - 1:] = sy * Tq[..., :0:-1, :]               # dj < 0
    F[..., :ny - 1, :nx - 1] = sx * sy * Tq[..., :0:-1, :0:-1]      # both < 0
    return F


def dense_matrix_layered(Tq, dsigma):
    """A = I - K D with K[(p,c),(q,c')] = T_pq(i-i', j-j'; k, k'); rows/cols (component, z, y, x)."""
    _, _, nz, _, ny, nx = Tq.shape
    N = nx * ny * nz
    F = expand_table(Tq)
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    iz, iy, ix = iz.ravel(), iy.ravel(), ix.ravel()
    dj = iy[:, None] - iy[None, :] + ny - 1
    di = ix[:, None] - ix[None, :] + nx - 1
    K = F[:, :, iz[:, None], iz[None, :], dj, di]  # (3, 3, N, N)
    Kmat = K.transpose(0, 2, 1, 3).reshape(3 * N, 3 * N)
    D = np.zeros((3 * N, 3 * N))
    ds = dsigma.reshape(N, 3, 3)
    for p in range(3):
        for q in range(3):
            D[p * N + np.arange(N), q * N + np.arange(N)] = ds[:, p, q]
    return np.eye(3 * N) - Kmat @ D


def layered_spectra(Tq):
    """fft2 over (dj, di) of the circulant embedding on (2ny, 2nx) -- offset d at index
    d mod 2n, the unused slot n set to 0 (as reading R5) -- of every (p, q, k, k') plane.
    Returns (3, 3, nz, nz, 2ny, 2nx)."""
    _, _, nz, _, ny, nx = Tq.shape
    F = expand_table(Tq)
    C = np.zeros((3, 3, nz, nz, 2 * ny, 2 * nx), np.complex128)
    dj = np.arange(-(ny - 1), ny) % (2 * ny)
    di = np.arange(-(nx - 1), nx) % (2 * nx)
    C[..., dj[:, None], di[None, :]] = F
    return sfft.fft2(C, axes=(4, 5), workers=WORKERS)


def layered_scatter(Mhat, dsigma, E):
    """G (dsigma E): pad J in x and y, fft2, Y[p,k] = sum_{q,k'} M[p,q,k,k'] J[q,k'] per
    horizontal wavenumber, ifft2, crop."""
    _, nz, ny, nx = E.shape
    J = np.einsum("zyxpq,qzyx->pzyx", dsigma, E)
    Jp = np.zeros((3, nz, 2 * ny, 2 * nx), np.complex128)
    Jp[:, :, :ny, :nx] = J
    Jh = sfft.fft2(Jp, axes=(2, 3), workers=WORKERS)
    Yh = np.einsum("pqkluv,qluv->pkuv", Mhat, Jh)
    return sfft.ifft2(Yh, axes=(2, 3), workers=WORKERS)[:, :, :ny, :nx]


class LayeredOperator:
    """Matrix-free A = I - G dsigma over a layered background (one rectangular domain)."""

    def __init__(self, Tq, dsigma):
        self.n = (Tq.shape[5], Tq.shape[4], Tq.shape[2])
        self.dsigma = dsigma
        self.Mhat = layered_spectra(Tq)

    def scatter(self, E):
        return layered_scatter(self.Mhat, self.dsigma, E)

    def __call__(self, E):
        return E - self.scatter(E)


def direct_rows_layered(Tq, dsigma, E, cells, identity=True):
    """(I - G dsigma) E at output cells (ix, iy, iz) by the literal sum over every source cell
    with the (mirror-expanded) table, R17: O(N) per output cell, any grid size."""
    _, _, nz, _, ny, nx = Tq.shape
    J = np.einsum("zyxpq,qzyx->pzyx", dsigma, E)  # (3, nz, ny, nx)
    sx = np.outer(SX, SX)
    sy = np.outer(SY, SY)
    out = np.zeros((len(cells), 3), np.complex128)
    ii = np.arange(nx)
    jj = np.arange(ny)
    for t, (cx, cy, cz) in enumerate(cells):
        di = cx - ii  # (nx,) offsets observer - source
        dj = cy - jj
        # T_pq(di, dj; cz, k') for all sources, by the mirror rules of R18
        Tk = Tq[:, :, cz]  # (3, 3, nz, ny, nx)
        A = Tk[:, :, :, np.abs(dj)[:, None], np.abs(di)[None, :]]  # (3, 3, nz, ny, nx)
        fx = np.where(di < 0, 1.0, 0.0)[None, None, None, None, :]
        fy = np.where(dj < 0, 1.0, 0.0)[None, None, None, :, None]
        A = A * np.where(fx > 0, sx[:, :, None, None, None], 1.0) * np.where(fy > 0, sy[:, :, None, None, None], 1.0)
        # odd components vanish at zero offset (R18)
        A = A * np.where((di == 0)[None, None, None, None, :], (sx > 0)[:, :, None, None, None], 1.0)
        A = A * np.where((dj == 0)[None, None, None, :, None], (sy > 0)[:, :, None, None, None], 1.0)
        s = np.einsum("pqzyx,qzyx->p", A, J)
        out[t] = (E[:, cz, cy, cx] if identity else 0.0) - s
    return out


def box_table(Tq, box):
    """The table of the diagonal block of box (i0,i1,j0,j1,k0,k1): offsets below its
    extents and layer indices inside its z-range (Eq. 15 for the layered kernel)."""
    i0, i1, j0, j1, k0, k1 = box
    return np.ascontiguousarray(Tq[:, :, k0:k1, k0:k1, :j1 - j0, :i1 - i0])


def homogeneous_table(n, h, k0, sigma_b):
    """Degenerate (equal-layer) table: T_pq(di, dj; k, k') = K_pq(di, dj, k - k') from the
    homogeneous kernel (Eq. 5 midpoint samples + reading R3 self term)."""
    nx, ny, nz = n
    K = physics.kernel_offsets(n, h, k0, sigma_b)  # [dz+nz-1, dy+ny-1, dx+nx-1, p, q]
    k = np.arange(nz)
    dz = k[:, None] - k[None, :] + nz - 1  # (nz, nz)
    Kq = K[:, ny - 1:, nx - 1:]  # dy, dx >= 0
    T = Kq[dz]  # (nz, nz, ny, nx, 3, 3)
    return np.ascontiguousarray(T.transpose(4, 5, 0, 1, 2, 3))


def random_table(n, rng, scale=0.05):
    """Arbitrary complex quadrant table (mirror rules implied by the storage, R18)."""
    nx, ny, nz = n
    shape = (3, 3, nz, nz, ny, nx)
    return scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def background_per_layer(n, origin, h, sigma_layers, z_iface):
    """sigma_b at each cell layer k: layer l holds centroids z with z_iface[l-1] <= z <
    z_iface[l] (layers bottom to top)."""
    nz = n[2]
    z = origin[2] + h[2] * np.arange(nz)
    idx = np.searchsorted(np.asarray(z_iface, np.float64), z, side="right")
    return np.asarray(sigma_layers, np.float64)[idx]


def contrast_layered(sigma, sigma_bz):
    """dsigma = sigma - sigma_b(z_k) I per cell (P:48 with a z-dependent background)."""
    return np.asarray(sigma, np.float64) - np.asarray(sigma_bz)[:, None, None, None, None] * np.eye(3)


def receiver_coupling(E, dsigma, e0rx, h0, dv, omega):
    """m_r . H at a receiver dipole by reciprocity (R17 receivers): h0 + (i omega mu0)^-1
    sum_c E0_{m_r}(r_c) . (dsigma_c E_c) dv, with E0_{m_r} the caller-supplied background
    field of the unit receiver dipole (3, nz, ny, nx) and h0 = m_r . H0."""
    J = np.einsum("zyxpq,qzyx->pzyx", dsigma, E)
    return h0 + np.sum(e0rx * J) * dv / (1j * omega * physics.MU0)


class LayeredDDSystem:
    """The block pieces of Eq. 15 for a layered table: A (full domain) and A_ii (diagonal
    blocks from ``box_table``); same interface as dd.DDSystem (coupling by a full-domain
    convolution of the source restricted to box j, restricted to box i)."""

    def __init__(self, Tq, dsigma, boxes):
        from . import dd
        self.n = (Tq.shape[5], Tq.shape[4], Tq.shape[2])
        dd.check_partition(self.n, boxes)
        self.boxes = list(boxes)
        self.A = LayeredOperator(Tq, dsigma)
        self.Aii = [LayeredOperator(box_table(Tq, b), dsigma[dd.box_slices(b)[1:]]) for b in boxes]

    def coupling(self, i, j, E):
        from . import dd
        Ej = np.zeros_like(E)
        Ej[dd.box_slices(self.boxes[j])] = E[dd.box_slices(self.boxes[j])]
        return self.A.scatter(Ej)[dd.box_slices(self.boxes[i])]
