"""Pins of oracle/operator.py: the FFT convolution of Eq. 10 against the literal sum of
Eq. 3 (dense matrix and direct rows), special cases, and the spectral parities the CUDA
path exploits (CPU, -m "not gpu")."""

import numpy as np
import pytest

from oracle import physics, operator as op


def _rand_case(n, seed, sigma_b=0.3, freq=4e5, h=(0.2, 0.25, 0.15)):
    rng = np.random.default_rng(seed)
    nx, ny, nz = n
    A = rng.standard_normal((nz, ny, nx, 3, 3))
    ds = 0.5 * (A + np.swapaxes(A, -1, -2))
    E = rng.standard_normal((3, nz, ny, nx)) + 1j * rng.standard_normal((3, nz, ny, nx))
    k0 = physics.wavenumber(sigma_b, freq)
    return h, k0, sigma_b, ds, E


@pytest.mark.parametrize("n", [(4, 3, 5), (2, 2, 2), (1, 4, 2), (6, 5, 3)])
def test_fft_apply_equals_dense_matrix(n):
    h, k0, sb, ds, E = _rand_case(n, 1)
    A = op.dense_matrix(n, h, k0, sb, ds)
    y_dense = (A @ E.ravel()).reshape(E.shape)
    y_fft = op.Operator(n, h, k0, sb, ds)(E)
    assert np.linalg.norm(y_fft - y_dense) / np.linalg.norm(y_dense) < 1e-13


def test_direct_rows_equal_dense_matrix():
    n = (5, 4, 3)
    h, k0, sb, ds, E = _rand_case(n, 2)
    A = op.dense_matrix(n, h, k0, sb, ds)
    y = (A @ E.ravel()).reshape(E.shape)
    cells = [(0, 0, 0), (4, 3, 2), (2, 1, 1)]
    yd = op.direct_rows(n, h, k0, sb, ds, E, cells)
    for t, (x, yy, z) in enumerate(cells):
        assert np.abs(yd[t] - y[:, z, yy, x]).max() < 1e-13 * np.abs(y).max()


def test_zero_contrast_is_identity_bitwise():
    n = (4, 4, 4)
    h, k0, sb, ds, E = _rand_case(n, 3)
    y = op.Operator(n, h, k0, sb, np.zeros_like(ds))(E)
    assert np.array_equal(y, E)


def test_delta_source_gives_green_column():
    """A unit contrast source in one cell and component returns K(c - c') column q at every
    cell (Eq. 10 reproduces the Green matrix column)."""
    n = (4, 3, 5)
    h, k0, sb, _, _ = _rand_case(n, 4)
    nx, ny, nz = n
    ds = np.zeros((nz, ny, nx, 3, 3))
    ds[...] = np.eye(3)
    src = (1, 2, 3)  # (x, y, z)
    q = 2
    E = np.zeros((3, nz, ny, nx), complex)
    E[q, src[2], src[1], src[0]] = 1.0
    G = op.Operator(n, h, k0, sb, ds).scatter(E)
    K = physics.kernel_offsets(n, h, k0, sb)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                col = K[z - src[2] + nz - 1, y - src[1] + ny - 1, x - src[0] + nx - 1][:, q]
                assert np.abs(G[:, z, y, x] - col).max() < 1e-14 * np.abs(K).max()


def test_linearity_and_relres_special_cases():
    n = (4, 4, 2)
    h, k0, sb, ds, E1 = _rand_case(n, 5)
    E2 = np.roll(E1, 1, axis=1) * (0.3 - 0.2j)
    A = op.Operator(n, h, k0, sb, ds)
    a, b = 1.3 - 0.7j, -0.4 + 2j
    lhs = A(a * E1 + b * E2)
    rhs = a * A(E1) + b * A(E2)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-14
    # Eq. 9: E = 0 gives e = 1
    assert op.relative_residual(A, np.zeros_like(E1), E1) == 1.0


def test_green_spectrum_axis_parities():
    """K_pq is even in each axis except xy (odd in x,y), xz (odd in x,z), yz (odd in y,z);
    so F[G_pq](2n - k) = +-F[G_pq](k) per axis -- the octant storage the CUDA path uses."""
    n = (4, 6, 2)
    h, k0, sb, _, _ = _rand_case(n, 6)
    Gh = op.green_spectra(n, h, k0, sb)
    odd = {(0, 1): (1, 1, 0), (0, 2): (1, 0, 1), (1, 2): (0, 1, 1)}
    scale = np.abs(Gh).max()
    for p in range(3):
        for q in range(3):
            ox, oy, oz = odd.get((min(p, q), max(p, q)), (0, 0, 0))
            G = Gh[p, q]
            fx = G[:, :, (-np.arange(2 * n[0])) % (2 * n[0])]
            assert np.abs(fx - (-1) ** ox * G).max() < 1e-13 * scale
            fy = G[:, (-np.arange(2 * n[1])) % (2 * n[1]), :]
            assert np.abs(fy - (-1) ** oy * G).max() < 1e-13 * scale
            fz = G[(-np.arange(2 * n[2])) % (2 * n[2]), :, :]
            assert np.abs(fz - (-1) ** oz * G).max() < 1e-13 * scale
            assert np.abs(Gh[p, q] - Gh[q, p]).max() == 0.0
