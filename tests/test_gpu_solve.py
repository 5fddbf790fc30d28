"""GPU parity of the solvers (A6 GMRES, A7-A9 DD Algorithm 1) and receivers (A11) against
the CPU oracle.  Fields and receiver voltages: relative error <= 1e-6 at solver
tolerance 1e-9 (BASELINE.json north_star); truth = dense LU (8^3 grids) or the oracle's
GMRES at 1e-12."""

import numpy as np
import pytest

from ie_workloads import make_config
from oracle import physics, operator as op, receivers as orx
from oracle.gmres import gmres
from gpu_helpers import gpu_ctx, oracle_setup, rel

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-6


def _lu_truth(cfg, sigma):
    k0, ds, E0 = oracle_setup(cfg, sigma)
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    X = np.stack([np.linalg.solve(A, e.ravel()).reshape(e.shape) for e in E0])
    return k0, ds, E0, X


def _field(cfg, ns):
    import torch
    nx, ny, nz = cfg.n
    return torch.empty((ns, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")


def test_c1_full_gmres_vs_dense_lu_every_cell():
    import paper_2306_17537_b200 as ie
    cfg = make_config("c1")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, "full", outer_tol=1e-10, restart=30, max_iters=500)
    assert rel(e.cpu().numpy(), X) < FIELD_TOL
    assert st["e_final"] <= 1e-10


def test_solve_subdomain_matches_oracle_gmres_and_lu():
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mini")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    b = torch.from_numpy(E0).cuda()
    x = b.clone()
    stats, _ = ie.ie_solve_subdomain(ctx, b, x, tol=1e-9, restart=10, max_iters=2000)
    assert stats[0]["converged"] and stats[0]["relres_true"] <= 1e-9
    assert rel(x.cpu().numpy(), X) < FIELD_TOL
    # oracle GMRES iteration count on the same system (loose: +-10%, SURVEY 8c uniqueness)
    _, info = gmres(op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds), E0[0], x0=E0[0], tol=1e-9, restart=10)
    assert abs(stats[0]["iters"] - info["iters"]) <= max(2, 0.1 * info["iters"])


def test_solve_subdomain_box_and_zero_rhs():
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mini")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, _ = _lu_truth(cfg, sigma)
    box = (0, 8, 0, 8, 4, 8)
    Ab = op.dense_matrix((8, 8, 4), cfg.hvec, k0, cfg.sigma_b, ds[4:8])
    rng = np.random.default_rng(5)
    bb = rng.standard_normal((2, 3, 4, 8, 8)) + 1j * rng.standard_normal((2, 3, 4, 8, 8))
    bb[1] = 0.0
    b = torch.from_numpy(bb).cuda()
    x = torch.zeros_like(b)
    stats, _ = ie.ie_solve_subdomain(ctx, b, x, tol=1e-10, restart=30, box=box)
    ref = np.linalg.solve(Ab, bb[0].ravel()).reshape(bb[0].shape)
    assert rel(x.cpu().numpy()[0], ref) < FIELD_TOL
    assert np.all(x.cpu().numpy()[1] == 0) and stats[1]["converged"] and stats[1]["iters"] == 0


@pytest.mark.parametrize("name", ["c2mini", "c3mini", "c5mini"])
@pytest.mark.parametrize("scheme", ["jacobi", "gauss_seidel"])
def test_dd_converges_to_dense_lu(name, scheme):
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    e = _field(cfg, len(cfg.sources))
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=cfg.restart)
    assert st["e_final"] <= 1e-9
    assert rel(e.cpu().numpy(), X) < FIELD_TOL
    # receivers: H at the config's receivers vs the oracle on the LU field
    H, V = ie.ie_receiver_fields(ctx, e, np.array(cfg.receivers))
    for s, (pos, m) in enumerate(cfg.sources):
        Href = orx.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, X[s], cfg.receivers, pos, m)
        assert rel(H[s], Href) < FIELD_TOL
        Vref = 1j * 2 * np.pi * cfg.freq * physics.MU0 * Href
        assert rel(V[s], Vref) < FIELD_TOL


def test_dd_gs_single_sweep_matches_oracle_forward_substitution():
    """One GS sweep with tight inner tolerance = Appendix A forward substitution."""
    import paper_2306_17537_b200 as ie
    from oracle import dd
    cfg = make_config("c2mini")
    boxes = [(0, 8, 0, 8, 0, 2), (0, 8, 0, 8, 2, 4), (0, 8, 0, 8, 4, 8)]
    ctx, sigma = gpu_ctx(cfg, boxes=boxes, restart=60)  # workspace sized for the restart used below
    k0, ds, E0, _ = _lu_truth(cfg, sigma)
    A = op.dense_matrix(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    blocks, ids = dd.dense_blocks(A, cfg.n, boxes)
    ref = dd.dense_gs_sweep(blocks, [E0[0].ravel()[i] for i in ids], [E0[0].ravel()[i] for i in ids])
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, "gauss_seidel", boxes=boxes, outer_tol=1e-30, adaptive=False,
                        inner_tol_fixed=1e-13, max_sweeps=1, restart=60, check=False)
    # outer_tol 1e-30 is out of reach, so stopping at max_sweeps=1 reports NOT_CONVERGED (R16)
    assert ie.STATUS[st["status"]] == "IE_ERR_NOT_CONVERGED" and st["sweeps"] == 1, (ie.STATUS.get(st["status"]),
                                                                           ctx.last_error())
    got = e.cpu().numpy()[0].ravel()
    for b in range(3):
        assert np.linalg.norm(got[ids[b]] - ref[b]) < 1e-10 * np.linalg.norm(E0)


def test_dd_zero_contrast_zero_sweeps():
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mini")
    sig = np.zeros((8, 8, 8, 3, 3)) + cfg.sigma_b * np.eye(3)
    ctx, _ = gpu_ctx(cfg, sigma=sig)
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, "jacobi", boxes=cfg.boxes, outer_tol=1e-12)
    assert st["sweeps"] == 0
    _, _, E0 = oracle_setup(cfg, sig)
    assert np.array_equal(e.cpu().numpy(), E0) or rel(e.cpu().numpy(), E0) < 1e-15
    H, _ = ie.ie_receiver_fields(ctx, e, np.array(cfg.receivers))
    k0 = physics.wavenumber(cfg.sigma_b, cfg.freq)
    H0 = physics.incident_H(np.array(cfg.receivers), cfg.sources[0][0], cfg.sources[0][1], k0)
    assert rel(H[0], H0) < 1e-14


@pytest.mark.parametrize("scheme", ["full", "jacobi", "gauss_seidel"])
def test_c2mod_solves_match_oracle_gmres(scheme):
    """c2mod (the c2 geometry, 32^3, 2 z-boxes, moderate contrast): GPU at tol 1e-9 vs oracle
    full-domain GMRES at 1e-12."""
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mod")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0 = oracle_setup(cfg, sigma)
    Aop = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    Xref, info = gmres(Aop, E0[0], x0=E0[0], tol=1e-12, restart=30, max_iters=3000)
    assert info["converged"]
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=30, max_sweeps=300)
    assert rel(e.cpu().numpy()[0], Xref) < FIELD_TOL
    H, _ = ie.ie_receiver_fields(ctx, e, np.array(cfg.receivers))
    Href = orx.receiver_H(cfg.n, cfg.hvec, cfg.origin, k0, cfg.sigma_b, ds, Xref, cfg.receivers, *cfg.sources[0])
    assert rel(H[0], Href) < FIELD_TOL


@pytest.mark.parametrize("name", ["c1", "c2mini", "c3mini", "c5mini"])
@pytest.mark.parametrize("scheme", ["full", "jacobi", "gauss_seidel"])
def test_contraction_preconditioned_solves_match_dense_lu(name, scheme):
    """Right preconditioner P = 2 sigma_b (sigma + sigma_b I)^-1 (contraction IE):
    the same discrete solution (dense LU) and the same Eq. 9 residual."""
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    e = _field(cfg, len(cfg.sources))
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=cfg.restart, precond=1)
    assert st["e_final"] <= 1e-9
    assert rel(e.cpu().numpy(), X) < FIELD_TOL


def test_contraction_preconditioned_subdomain_solve_on_a_box():
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mini")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, _ = _lu_truth(cfg, sigma)
    box = (0, 8, 0, 8, 2, 6)
    Ab = op.dense_matrix((8, 8, 4), cfg.hvec, k0, cfg.sigma_b, ds[2:6])
    rng = np.random.default_rng(8)
    bb = rng.standard_normal((1, 3, 4, 8, 8)) + 1j * rng.standard_normal((1, 3, 4, 8, 8))
    b = torch.from_numpy(bb).cuda()
    x = b.clone()
    stats, _ = ie.ie_solve_subdomain(ctx, b, x, tol=1e-10, restart=30, box=box, precond=1)
    assert stats[0]["converged"] and stats[0]["relres_true"] <= 1e-10
    ref = np.linalg.solve(Ab, bb[0].ravel()).reshape(bb[0].shape)
    assert rel(x.cpu().numpy()[0], ref) < FIELD_TOL


@pytest.mark.parametrize("scheme", ["full", "gauss_seidel"])
def test_c2mod_preconditioned_matches_oracle_gmres(scheme):
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mod")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0 = oracle_setup(cfg, sigma)
    Aop = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    Xref, info = gmres(Aop, E0[0], x0=E0[0], tol=1e-12, restart=30, max_iters=3000)
    assert info["converged"]
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=30, max_sweeps=300, precond=1)
    assert rel(e.cpu().numpy()[0], Xref) < FIELD_TOL


@pytest.mark.parametrize("name", ["c2mini", "c3mini", "c5mini"])
@pytest.mark.parametrize("scheme", ["fgmres_jacobi", "fgmres_gauss_seidel"])
@pytest.mark.parametrize("precond", [0, 1])
def test_krylov_accelerated_dd_matches_dense_lu(name, scheme, precond):
    """FGMRES right-preconditioned by one block-Jacobi / block-GS sweep
    reaches the dense LU solution."""
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    e = _field(cfg, len(cfg.sources))
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=cfg.restart,
                        inner_tol_fixed=1e-2, max_sweeps=100, precond=precond)
    assert st["e_final"] <= 1e-9
    assert rel(e.cpu().numpy(), X) < FIELD_TOL


@pytest.mark.parametrize("scheme", ["fgmres_jacobi", "fgmres_gauss_seidel"])
def test_c2mod_krylov_dd_matches_oracle_gmres(scheme):
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mod")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0 = oracle_setup(cfg, sigma)
    Aop = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    Xref, info = gmres(Aop, E0[0], x0=E0[0], tol=1e-12, restart=30, max_iters=3000)
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=30, inner_tol_fixed=1e-2,
                        max_sweeps=100)
    assert rel(e.cpu().numpy()[0], Xref) < FIELD_TOL


def _tall_cfg(n, boxes):
    """Tall grids whose z-pass runs the TMEM kernels (2nz = 256, 128), z-split sub-domains so the
    Gauss-Seidel coupling applies have z-restricted sources; smooth anisotropic contrast of the
    c2mod kind (moderate, so the oracle GMRES converges quickly)."""
    from ie_workloads import Config

    def sig(rng, cfg):
        nx, ny, nz = cfg.n
        A = rng.standard_normal((nz, ny, nx, 3, 3)) * 0.05
        return 0.5 * (A + np.swapaxes(A, -1, -2)) + (cfg.sigma_b * 1.5) * np.eye(3)

    return Config("tall", n, 0.2, 0.3, 4e5, 11, sig,
                  sources=[(np.array([0.013, 0.021, 0.017]), np.array([0.2, -0.3, 1.0]))],
                  boxes=boxes, restart=30)


@pytest.mark.parametrize("n,boxes", [
    ((8, 8, 128), [(0, 8, 0, 8, 0, 64), (0, 8, 0, 8, 64, 128)]),
    ((16, 16, 64), [(0, 16, 0, 16, 0, 32), (0, 16, 0, 16, 32, 48), (0, 16, 0, 16, 48, 64)]),
])
@pytest.mark.parametrize("scheme", ["jacobi", "gauss_seidel"])
def test_tall_grid_dd_matches_oracle_gmres(n, boxes, scheme):
    """DD on 2nz = 256 / 128 grids (TMEM z-pass with z-restricted coupling sources; unequal
    z-boxes) at tol 1e-9 vs the oracle's full-domain GMRES at 1e-12."""
    import paper_2306_17537_b200 as ie
    cfg = _tall_cfg(n, boxes)
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0 = oracle_setup(cfg, sigma)
    Aop = op.Operator(cfg.n, cfg.hvec, k0, cfg.sigma_b, ds)
    Xref, info = gmres(Aop, E0[0], x0=E0[0], tol=1e-12, restart=30, max_iters=3000)
    assert info["converged"]
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-9, restart=30, max_sweeps=300)
    assert st["e_final"] <= 1e-9
    assert rel(e.cpu().numpy()[0], Xref) < FIELD_TOL


@pytest.mark.parametrize("scheme", ["full", "gauss_seidel", "jacobi"])
def test_warm_start_and_preconditioner_calls(scheme):
    """ie_solve_dd_warm starts from the caller's iterate (a converged field: 0 sweeps / iterations,
    the field unchanged); ie_solve_dd starts from E0 whatever e_dev holds; ie_set_preconditioner
    rejects unknown kinds and kind 1 reaches the same solution."""
    import torch
    import paper_2306_17537_b200 as ie
    cfg = make_config("c2mini")
    ctx, sigma = gpu_ctx(cfg)
    k0, ds, E0, X = _lu_truth(cfg, sigma)
    e = _field(cfg, 1)
    st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-10, restart=30, max_sweeps=300)
    assert rel(e.cpu().numpy(), X) < FIELD_TOL
    e_conv = e.clone()
    st2 = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-10, restart=30, init_from_e=True,
                         min_iters=0)
    assert st2["total_inner_iters"] == 0 and st2["sweeps"] == 0
    assert torch.equal(e, e_conv)
    e.fill_(1e3)  # cold start ignores the content
    st3 = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-10, restart=30, max_sweeps=300)
    assert st3["total_inner_iters"] == st["total_inner_iters"] and rel(e.cpu().numpy(), X) < FIELD_TOL
    with pytest.raises(ie.IEError):
        ie.ie_set_preconditioner(ctx, 2)
    ie.ie_set_preconditioner(ctx, 1)
    st4 = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-10, restart=30, max_sweeps=300, precond=1)
    assert rel(e.cpu().numpy(), X) < FIELD_TOL and st4["e_final"] <= 1e-10


@pytest.mark.parametrize("name,scheme,precond", [("c2mini", "full", 0), ("c2mini", "jacobi", 1),
                                                 ("c5mini", "gauss_seidel", 0), ("c3mini", "fgmres_jacobi", 0)])
def test_device_side_arnoldi_matches_dense_lu(name, scheme, precond):
    """The opt-in device-side Arnoldi recurrences (IE_GMRES_DEVICE=1 at context creation: Hessenberg
    column, DGKS test, Givens rotations and stop rule on the device, look-ahead 1) reach the same
    solution as dense LU; iteration counts within one per solve of the host-recurrence path."""
    import os
    import paper_2306_17537_b200 as ie
    cfg = make_config(name)
    out = []
    for dev in ("1", "0"):
        os.environ["IE_GMRES_DEVICE"] = dev
        try:
            ctx, sigma = gpu_ctx(cfg)
        finally:
            os.environ.pop("IE_GMRES_DEVICE", None)
        k0, ds, E0, X = _lu_truth(cfg, sigma)
        e = _field(cfg, len(E0))
        st = ie.ie_solve_dd(ctx, e, scheme, boxes=cfg.boxes, outer_tol=1e-10, restart=30, max_sweeps=300,
                            inner_tol_fixed=1e-2 if scheme.startswith("fgmres") else 1e-6, precond=precond)
        assert st["e_final"] <= 1e-10
        assert rel(e.cpu().numpy(), X) < FIELD_TOL
        out.append(st)
    assert abs(out[0]["total_inner_iters"] - out[1]["total_inner_iters"]) <= max(2, out[1]["total_inner_iters"] // 50)
