"""Pins of oracle/layered.py (layered-table operator, readings R17-R19): the mirror rules
against the homogeneous kernel, FFT path vs brute-force dense assembly on arbitrary
tables, the degenerate table against the Eq. 10 operator, the box (diagonal-block) table,
the reciprocity receiver form, and DD on a layered table vs dense LU."""

import numpy as np
import pytest

from oracle import physics, operator as op, layered as lay, dd


def _hom(n, h=0.25, sigma_b=0.7, f=2e5):
    k0 = physics.wavenumber(sigma_b, f)
    return k0, lay.homogeneous_table(n, (h, h, h), k0, sigma_b), (h, h, h), sigma_b


def _field(rng, n):
    nx, ny, nz = n
    return rng.standard_normal((3, nz, ny, nx)) + 1j * rng.standard_normal((3, nz, ny, nx))


def _dsig(rng, n, s=0.4):
    nx, ny, nz = n
    A = rng.standard_normal((nz, ny, nx, 3, 3)) * s
    return 0.5 * (A + np.swapaxes(A, -1, -2))


def test_mirror_rules_reproduce_the_homogeneous_kernel_at_negative_offsets():
    """expand_table(quadrant of K) must equal K at every offset: checks the sign vectors
    sx = (-1,1,1), sy = (1,-1,1) against the closed-form kernel (Eq. 5)."""
    n = (4, 3, 3)
    k0, Tq, h, sb = _hom(n)
    F = lay.expand_table(Tq)  # (3,3,nz,nz,2ny-1,2nx-1)
    K = physics.kernel_offsets(n, h, k0, sb)  # [dz, dy, dx, p, q]
    nx, ny, nz = n
    for k in range(nz):
        for kp in range(nz):
            ref = K[k - kp + nz - 1].transpose(2, 3, 0, 1)  # (3,3,2ny-1,2nx-1)
            assert np.array_equal(F[:, :, k, kp], ref)


@pytest.mark.parametrize("n", [(4, 4, 3), (2, 4, 2), (8, 2, 2)])
def test_fft_path_equals_dense_assembly_on_arbitrary_tables(n):
    rng = np.random.default_rng(11)
    Tq = lay.random_table(n, rng)
    ds = _dsig(rng, n)
    x = _field(rng, n)
    A = lay.dense_matrix_layered(Tq, ds)
    y_dense = (A @ x.ravel()).reshape(x.shape)
    y_fft = lay.LayeredOperator(Tq, ds)(x)
    assert np.linalg.norm(y_fft - y_dense) < 1e-13 * np.linalg.norm(y_dense)


def test_dense_assembly_is_not_blind_to_k_kprime_order():
    """An arbitrary (non-Toeplitz) table: swapping k and k' must change the operator."""
    n = (2, 2, 3)
    rng = np.random.default_rng(3)
    Tq = lay.random_table(n, rng)
    ds = _dsig(rng, n)
    A1 = lay.dense_matrix_layered(Tq, ds)
    A2 = lay.dense_matrix_layered(np.ascontiguousarray(Tq.swapaxes(2, 3)), ds)
    assert np.abs(A1 - A2).max() > 1e-3


@pytest.mark.parametrize("n", [(8, 4, 4), (4, 8, 8)])
def test_degenerate_table_equals_the_homogeneous_operator(n):
    k0, Tq, h, sb = _hom(n)
    rng = np.random.default_rng(5)
    ds = _dsig(rng, n)
    x = _field(rng, n)
    y_lay = lay.LayeredOperator(Tq, ds)(x)
    y_hom = op.Operator(n, h, k0, sb, ds)(x)
    assert np.linalg.norm(y_lay - y_hom) < 1e-13 * np.linalg.norm(y_hom)
    A_lay = lay.dense_matrix_layered(Tq, ds) if np.prod(n) <= 128 else None
    if A_lay is not None:
        assert np.abs(A_lay - op.dense_matrix(n, h, k0, sb, ds)).max() == 0.0


def test_box_table_gives_the_diagonal_block():
    n = (4, 2, 4)
    rng = np.random.default_rng(7)
    Tq = lay.random_table(n, rng)
    ds = _dsig(rng, n)
    A = lay.dense_matrix_layered(Tq, ds)
    box = (2, 4, 0, 2, 1, 3)
    Ab = lay.dense_matrix_layered(lay.box_table(Tq, box), ds[1:3, 0:2, 2:4])
    nx, ny, nz = n
    cells = [(z, y, x) for z in range(1, 3) for y in range(0, 2) for x in range(2, 4)]
    N = nx * ny * nz
    idx = np.array([[p * N + (z * ny + y) * nx + x for (z, y, x) in cells] for p in range(3)]).ravel()
    assert np.abs(A[np.ix_(idx, idx)] - Ab).max() < 1e-15


def test_background_per_layer_and_contrast():
    n, origin, h = (2, 2, 8), (0, 0, -3.5), (1, 1, 1)
    sb = lay.background_per_layer(n, origin, h, [1.0, 0.01, 1.0], [-2.0, 2.0])
    assert list(sb) == [1.0, 1.0, 0.01, 0.01, 0.01, 0.01, 1.0, 1.0]  # z = -3.5 .. 3.5
    sig = np.ones((8, 2, 2, 3, 3))
    ds = lay.contrast_layered(sig, sb)
    assert ds[2, 0, 0, 0, 0] == 0.99 and ds[0, 1, 1, 1, 1] == 0.0 and ds[0, 0, 0, 0, 1] == 1.0


def test_reciprocity_receiver_form_equals_direct_H_homogeneous():
    """receiver_coupling with the homogeneous E0 of the receiver dipole equals
    m_r . H of Eq. 4 (receivers.receiver_H) on a solved field."""
    from ie_workloads import make_config
    from oracle import receivers
    cfg = make_config("c2mini")
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    ds = physics.contrast(cfg.sigma(), cfg.sigma_b)
    src, m = cfg.sources[0]
    pts = physics.centroids(cfg.n, cfg.hvec, cfg.origin)
    E0 = np.moveaxis(physics.incident_E(pts, src, m, k0, cfg.freq), -1, 0)
    E = np.linalg.solve(op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds), E0.ravel()).reshape(E0.shape)
    rx, mr = np.array([0.05, -0.05, 0.85]), np.array([0.3, -1.0, 0.5])
    H = receivers.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, E, [rx], src, m)[0]
    e0rx = np.moveaxis(physics.incident_E(pts, rx, mr, k0, cfg.freq), -1, 0)
    h0 = mr @ physics.incident_H(rx, src, m, k0)
    v = lay.receiver_coupling(E, ds, e0rx, h0, cfg.h ** 3, physics.omega_of(cfg.freq))
    assert abs(v - mr @ H) < 1e-12 * abs(mr @ H)


@pytest.mark.parametrize("scheme", ["jacobi", "gauss_seidel"])
def test_layered_dd_converges_to_dense_lu(scheme):
    """A perturbed degenerate table (not Toeplitz in z) with 2 z-boxes: Algorithm 1 on the
    layered operator reaches the dense solution."""
    n = (4, 4, 4)
    k0, Tq, h, sb = _hom(n)
    rng = np.random.default_rng(9)
    Tq = Tq + lay.random_table(n, rng, scale=2e-3)
    ds = np.abs(_dsig(rng, n, 0.2))
    ds = 0.5 * (ds + np.swapaxes(ds, -1, -2))
    E0 = _field(rng, n)
    X = np.linalg.solve(lay.dense_matrix_layered(Tq, ds), E0.ravel()).reshape(E0.shape)
    boxes = [(0, 4, 0, 4, 0, 2), (0, 4, 0, 4, 2, 4)]
    sysl = lay.LayeredDDSystem(Tq, ds, boxes)
    E, st = dd.solve_dd(sysl, E0, scheme, outer_tol=1e-11, restart=30)
    assert st["converged"]
    assert np.linalg.norm(E - X) < 1e-8 * np.linalg.norm(X)


def test_spectrum_mirror_relation_on_arbitrary_tables():
    """M(2n - kx) = Dx M(kx) Dx and M(2n - ky) = Dy M(ky) Dy (D = diag of the mirror signs): the
    structure the GPU z-contraction relies on to serve 4 wavenumbers from one matrix."""
    n = (8, 4, 3)
    nx, ny, nz = n
    M = lay.layered_spectra(lay.random_table(n, np.random.default_rng(12)))
    for ix, iy in [(1, 1), (3, 2), (0, 3), (4, 0)]:
        a = M[..., iy, (2 * nx - ix) % (2 * nx)]
        b = np.einsum("p,q,pqkl->pqkl", lay.SX, lay.SX, M[..., iy, ix])
        assert np.abs(a - b).max() < 1e-15 * np.abs(M).max()
        a = M[..., (2 * ny - iy) % (2 * ny), ix]
        b = np.einsum("p,q,pqkl->pqkl", lay.SY, lay.SY, M[..., iy, ix])
        assert np.abs(a - b).max() < 1e-15 * np.abs(M).max()


def test_direct_rows_layered_equal_dense_assembly():
    n = (5, 4, 3)
    rng = np.random.default_rng(21)
    Tq = lay.random_table(n, rng)
    ds = _dsig(rng, n, 0.3)
    E = _field(rng, n)
    y = (lay.dense_matrix_layered(Tq, ds) @ E.ravel()).reshape(E.shape)
    cells = [(0, 0, 0), (4, 3, 2), (2, 1, 1), (3, 0, 2)]
    yd = lay.direct_rows_layered(Tq, ds, E, cells)
    for t, (x, yy, z) in enumerate(cells):
        assert np.abs(yd[t] - y[:, z, yy, x]).max() < 1e-13 * np.abs(y).max()


@pytest.mark.parametrize("scheme", ["jacobi", "gauss_seidel"])
def test_physical_layered_dd_converges_to_dense_lu(scheme):
    """The c4 recipe on 8^3 with the physical three-layer table (layered_green): Algorithm 1
    (2 x 2 boxes in x, y) reaches the dense LU solution, with E0 of the layered background."""
    from ie_workloads import make_config, layered_inputs as li
    cfg = make_config("c4lmini")
    med = li.medium(cfg)
    Tq = li.table(cfg, med)
    sbz = lay.background_per_layer(cfg.n, cfg.origin, cfg.hvec, *cfg.background())
    ds = lay.contrast_layered(cfg.sigma(), sbz)
    E0 = li.incident(cfg, med)[0]
    X = np.linalg.solve(lay.dense_matrix_layered(Tq, ds), E0.ravel()).reshape(E0.shape)
    E, st = dd.solve_dd(lay.LayeredDDSystem(Tq, ds, cfg.boxes), E0, scheme, outer_tol=1e-11, restart=30)
    assert st["converged"]
    assert np.linalg.norm(E - X) < 1e-8 * np.linalg.norm(X)
