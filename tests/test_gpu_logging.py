"""The moving-window logging pipeline on a small window: window
conductivity from the formation in the rotated frame, the axial transmitter's E0, GS-A on two
sub-domains along the hole, receiver fields -- against the oracle's dense LU solution and Eq. 4."""

import numpy as np
import pytest

from ie_workloads import logging as lg
from oracle import physics, operator as op, receivers as orx
from gpu_helpers import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("station", [1, 3])
@pytest.mark.parametrize("precond", [0, 1])
def test_window_station_matches_dense_lu(station, precond):
    import torch
    import paper_2306_17537_b200 as ie
    n, h = (16, 8, 8), 2.0
    nx, ny, nz = n
    origin, _ = lg.window_grid(n, h, behind=8.0)
    tx = lg.stations(5)[station]
    sig = lg.window_sigma(tx, n, h, behind=8.0)
    boxes = [(0, 8, 0, 8, 0, 8), (8, 16, 0, 8, 0, 8)]
    ctx = ie.ie_create(n, (h, h, h), origin, lg.SIGMA0, lg.FREQ)
    ie.ensure_workspace(ctx, boxes=boxes, nrhs=1, restart=30)
    ie.ie_set_contrast(ctx, torch.from_numpy(np.ascontiguousarray(sig)).cuda())
    txw, mw, rxw = lg.tool_in_window()
    ie.ie_set_source(ctx, txw[None], mw[None])
    e = torch.empty((1, 3, nz, ny, nx), dtype=torch.complex128, device="cuda")
    st = ie.ie_solve_dd(ctx, e, "gauss_seidel", boxes=boxes, outer_tol=1e-10, restart=30, max_sweeps=300,
                        precond=precond)
    assert st["e_final"] <= 1e-10
    k0 = physics.wavenumber(lg.SIGMA0, lg.FREQ)
    ds = physics.contrast(sig, lg.SIGMA0)
    pts = physics.centroids(n, (h, h, h), origin)
    E0 = np.moveaxis(physics.incident_E(pts, txw, mw, k0, lg.FREQ), -1, 0)
    X = np.linalg.solve(op.dense_matrix(n, (h, h, h), k0, lg.SIGMA0, ds), E0.ravel()).reshape(E0.shape)
    assert rel(e.cpu().numpy()[0], X) < 1e-6
    H, _ = ie.ie_receiver_fields(ctx, e, np.array(rxw))
    Href = orx.receiver_H(n, (h, h, h), origin, k0, lg.SIGMA0, ds, X, rxw, txw, mw)
    assert rel(H[0], Href) < 1e-6


def test_device_window_sigma_equals_the_host_recipe():
    """The device (torch) sampling of the formation in the window frame equals the numpy recipe
    (ie_workloads.logging.window_sigma) to roundoff on the window-1 shape at several stations."""
    for tx in lg.stations(4):
        a = lg.window_sigma(tx, (64, 32, 32), 0.25)
        b = lg.window_sigma_device(tx, (64, 32, 32), 0.25).cpu().numpy()
        assert np.abs(a - b).max() <= 1e-15 * np.abs(a).max()
