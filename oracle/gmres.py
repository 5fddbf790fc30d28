"""Restarted GMRES (Saad & Schultz 1986), the paper's linear solver.

Plain textbook algorithm: Arnoldi with modified Gram-Schmidt, complex Givens rotations,
least-squares update at convergence or restart.  Stopping rule (reading R8): stop when the
estimated ||b - A x|| / ||b|| <= tol (relative to ||b||, as Eq. 9 is relative to ||E0||);
at every restart and at exit the true residual is recomputed.  ``min_iters`` implements the
DD stall guard (reading R10).  Iteration count = number of A v products in Arnoldi.
"""

import numpy as np


def _dot(a, b):
    return np.vdot(a.ravel(), b.ravel())  # conj(a) . b


def _nrm(a):
    return float(np.linalg.norm(a.ravel()))


def gmres(A, b, x0=None, tol=1e-9, restart=30, max_iters=5000, min_iters=0):
    """Solve A x = b.  Returns (x, info) with info = dict(iters, restarts, converged,
    relres_est, relres_true, history)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    bnorm = _nrm(b)
    info = dict(iters=0, restarts=0, converged=False, relres_est=np.nan, relres_true=np.nan, history=[])
    if bnorm == 0.0:
        info.update(converged=True, relres_est=0.0, relres_true=0.0)
        return np.zeros_like(b), info
    r = b - A(x)
    beta = _nrm(r)
    info["relres_true"] = beta / bnorm
    if beta / bnorm <= tol and info["iters"] >= min_iters:
        info.update(converged=True, relres_est=beta / bnorm)
        return x, info
    while info["iters"] < max_iters:
        m = restart
        V = [r / beta]
        H = np.zeros((m + 1, m), np.complex128)
        cs = np.zeros(m, np.complex128)
        sn = np.zeros(m, np.complex128)
        g = np.zeros(m + 1, np.complex128)
        g[0] = beta
        k_done = 0
        done = False
        for k in range(m):
            w = A(V[k])
            if np.may_share_memory(w, V[k]):  # w is updated in place below
                w = w.copy()
            info["iters"] += 1
            for j in range(k + 1):  # modified Gram-Schmidt
                H[j, k] = _dot(V[j], w)
                w -= H[j, k] * V[j]
            H[k + 1, k] = _nrm(w)
            # apply previous rotations to the new column
            for j in range(k):
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -np.conj(sn[j]) * H[j, k] + np.conj(cs[j]) * H[j + 1, k]
                H[j, k] = t
            # new rotation zeroing H[k+1, k]
            a, c = H[k, k], H[k + 1, k]
            den = np.sqrt(abs(a) ** 2 + abs(c) ** 2)
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k] = a / den
                sn[k] = c / den
                cs[k], sn[k] = np.conj(cs[k]), np.conj(sn[k])
            H[k, k] = cs[k] * a + sn[k] * c
            H[k + 1, k] = 0.0
            g[k + 1] = -np.conj(sn[k]) * g[k]
            g[k] = cs[k] * g[k]
            k_done = k + 1
            est = abs(g[k + 1]) / bnorm
            info["history"].append(est)
            info["relres_est"] = est
            happy = _nrm(w) == 0.0
            if (est <= tol and info["iters"] >= min_iters) or info["iters"] >= max_iters or happy:
                done = True
                break
            V.append(w / _nrm(w))
        # least squares: H[:k,:k] y = g[:k]
        y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        for j in range(k_done):
            x += y[j] * V[j]
        r = b - A(x)
        beta = _nrm(r)
        info["relres_true"] = beta / bnorm
        if (beta / bnorm <= tol and info["iters"] >= min_iters) or beta == 0.0:
            info["converged"] = True
            return x, info
        if info["iters"] >= max_iters:
            return x, info
        info["restarts"] += 1
    return x, info
