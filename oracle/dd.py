"""Domain-decomposition fixed-point iteration, Algorithm 1 of the paper (oracle; test
infrastructure only).

Block system Eq. 14-16, splitting Eq. 17-18, block Gauss-Seidel
Eq. 19-22, block Jacobi Eq. 23-24, adaptive inner tolerance and
warm start (Algorithm 1).

Written deliberately naively: every coupling term G^(ij) dsigma^(j) E^(j)
is a separate full-grid FFT convolution of the source restricted to box j, then restricted
to box i.  Garbles in Algorithm 1 are resolved by readings R9-R12 in DESIGN.md:
e is recomputed after every sweep; the Jacobi sum excludes j = i (Eq. 24); E^0 := E^(0);
inner threshold = e/10 of the previous sweep; each sub-domain GMRES does >= 1 iteration.
"""

import numpy as np

from . import operator as op
from .gmres import gmres


def box_slices(box):
    """box = (i0, i1, j0, j1, k0, k1), half-open cell index ranges in x, y, z (Eq. 11)."""
    i0, i1, j0, j1, k0, k1 = box
    return (slice(None), slice(k0, k1), slice(j0, j1), slice(i0, i1))


def box_shape(box):
    i0, i1, j0, j1, k0, k1 = box
    return (i1 - i0, j1 - j0, k1 - k0)


def check_partition(n, boxes):
    nx, ny, nz = n
    cover = np.zeros((nz, ny, nx), np.int32)
    for b in boxes:
        cover[box_slices(b)[1:]] += 1
    if not np.all(cover == 1):
        raise ValueError("boxes must be a non-overlapping partition of the grid (Eq. 11)")


class DDSystem:
    """The block operator pieces of Eq. 15 for a given partition."""

    def __init__(self, n, h, k0, sigma_b, dsigma, boxes):
        check_partition(n, boxes)
        self.n, self.boxes = tuple(n), list(boxes)
        self.A = op.Operator(n, h, k0, sigma_b, dsigma)  # full-domain operator (Eq. 8)
        self.Aii = [op.Operator(box_shape(b), h, k0, sigma_b, dsigma[box_slices(b)[1:]]) for b in boxes]

    def coupling(self, i, j, E):
        """G^(ij) dsigma^(j) E^(j): field on box i due to the contrast source in box j (Eq. 13)."""
        Ej = np.zeros_like(E)
        Ej[box_slices(self.boxes[j])] = E[box_slices(self.boxes[j])]
        return self.A.scatter(Ej)[box_slices(self.boxes[i])]


def solve_dd(system, E0, scheme, outer_tol, adaptive=True, inner_tol_fixed=1e-6, inner_factor=0.1,
             restart=30, max_sweeps=200, inner_max_iters=2000, E_init=None):
    """Algorithm 1.  scheme in {"jacobi", "gauss_seidel"}.  Returns (E, stats)."""
    assert scheme in ("jacobi", "gauss_seidel")
    E = E0.copy() if E_init is None else E_init.copy()  # initialize: E^0 := E^(0)
    e = op.relative_residual(system.A, E, E0)  # Eq. 9
    stats = dict(sweeps=0, e_hist=[e], iters=[], total_inner_iters=0, converged=e <= outer_tol)
    grow = 0
    while e > outer_tol and stats["sweeps"] < max_sweeps:
        E_k = E.copy()  # iterate k (read by Jacobi; Eq. 24)
        its = []
        for i, bi in enumerate(system.boxes):
            src = E_k if scheme == "jacobi" else E  # GS uses the latest fields (Eq. 22)
            b = E0[box_slices(bi)].copy()  # E^(i,0)
            for j in range(len(system.boxes)):
                if j != i:
                    b = b + system.coupling(i, j, src)
            thr = e * inner_factor if adaptive else inner_tol_fixed  # threshold = e/10
            x0 = E_k[box_slices(bi)]  # initial guess = E^(i),k
            Ei, info = gmres(system.Aii[i], b, x0=x0, tol=thr, restart=restart,
                             max_iters=inner_max_iters, min_iters=1)
            E[box_slices(bi)] = Ei
            its.append(info["iters"])
        stats["sweeps"] += 1
        stats["iters"].append(its)
        stats["total_inner_iters"] += sum(its)
        e_new = op.relative_residual(system.A, E, E0)
        grow = grow + 1 if e_new > e else 0
        e = e_new
        stats["e_hist"].append(e)
        if grow >= 3:
            break
    stats["converged"] = e <= outer_tol
    stats["e_final"] = e
    return E, stats


# ---- Appendix A: dense forward substitution ---------------------------------

def box_index(n, box):
    """Flat unknown indices (component, z, y, x ordering) of the cells of ``box``."""
    nx, ny, nz = n
    N = nx * ny * nz
    idx = np.arange(3 * N).reshape(3, nz, ny, nx)
    return idx[box_slices(box)].ravel()


def dense_blocks(Adense, n, boxes):
    """A_ij blocks of Eq. A.1 from the dense matrix of Eq. 8."""
    ids = [box_index(n, b) for b in boxes]
    return [[Adense[np.ix_(ids[i], ids[j])] for j in range(len(boxes))] for i in range(len(boxes))], ids


def dense_gs_sweep(blocks, E0_blocks, E_blocks):
    """One block Gauss-Seidel sweep by forward substitution, Eqs. A.10-A.12 generalised:
    E_i^{k+1} = A_ii^{-1} [ R_i - sum_{j<i} A_ij E_j^{k+1} ],  R_i = E0_i - sum_{j>i} A_ij E_j^k."""
    M = len(blocks)
    out = [None] * M
    for i in range(M):
        R = E0_blocks[i].copy()
        for j in range(i + 1, M):
            R = R - blocks[i][j] @ E_blocks[j]
        for j in range(i):
            R = R - blocks[i][j] @ out[j]
        out[i] = np.linalg.solve(blocks[i][i], R)
    return out


def dense_gs_matrix_form(Adense, ids, E0, Ek):
    """Eq. A.5 / Eq. 20 directly: E^{k+1} = (D + L)^{-1} [E0 - U E^k] with dense D, L, U."""
    M = len(ids)
    n3 = Adense.shape[0]
    order = np.concatenate(ids)
    Ap = Adense[np.ix_(order, order)]
    sizes = [len(i) for i in ids]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    blockid = np.zeros(n3, np.int64)
    for b in range(M):
        blockid[offs[b]:offs[b + 1]] = b
    lower_or_diag = blockid[:, None] >= blockid[None, :]
    DL = np.where(lower_or_diag, Ap, 0.0)
    U = np.where(lower_or_diag, 0.0, Ap)
    rhs = E0[order] - U @ Ek[order]
    sol = np.linalg.solve(DL, rhs)
    out = np.empty_like(sol)
    out[order] = sol
    return out
