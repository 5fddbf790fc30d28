"""Input generators (ie_workloads): Appendix C rotation against rotation matrices and the
paper-derived worked examples; determinism; partitions; placement of sources."""

import json
import os

import numpy as np
import pytest

from ie_workloads import make_config, vti_tensor, haar_rotation, box_grid
from ie_workloads.configs import c4_stations

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_appendix_c_golden_examples():
    gold = json.load(open(os.path.join(GOLD, "appendix_c_examples.json")))
    for c in gold["cases"]:
        s = vti_tensor(c["sigma_h"], c["sigma_v"], c["theta"], c["phi"])
        assert np.abs(s - np.array(c["expect"])).max() < 1e-15


def test_appendix_c_equals_rotation_matrix_conjugation():
    """App. C == R diag(s_h, s_h, s_v) R^T with R = R_z(phi) R_y(theta): 100 draws;
    trace 2 s_h + s_v; eigenvalues {s_h, s_h, s_v}."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        sh, sv = rng.uniform(0.01, 5, 2)
        th, ph = rng.uniform(0, np.pi), rng.uniform(0, 2 * np.pi)
        Ry = np.array([[np.cos(th), 0, np.sin(th)], [0, 1, 0], [-np.sin(th), 0, np.cos(th)]])
        Rz = np.array([[np.cos(ph), -np.sin(ph), 0], [np.sin(ph), np.cos(ph), 0], [0, 0, 1]])
        R = Rz @ Ry
        ref = R @ np.diag([sh, sh, sv]) @ R.T
        s = vti_tensor(sh, sv, th, ph)
        assert np.abs(s - ref).max() < 1e-12
        assert abs(np.trace(s) - (2 * sh + sv)) < 1e-12
        assert np.abs(np.sort(np.linalg.eigvalsh(s)) - np.sort([sh, sh, sv])).max() < 1e-10


def test_haar_rotation_is_rotation():
    rng = np.random.default_rng(1)
    for _ in range(20):
        Q = haar_rotation(rng)
        assert np.abs(Q @ Q.T - np.eye(3)).max() < 1e-14
        assert abs(np.linalg.det(Q) - 1) < 1e-14


@pytest.mark.parametrize("name", ["c1", "c2", "c2mini", "c3mini", "c5mini", "c3h"])
def test_configs_deterministic_symmetric_and_placed(name):
    cfg = make_config(name)
    s1, s2 = cfg.sigma(), cfg.sigma()
    assert np.array_equal(s1, s2)
    assert s1.shape == (cfg.n[2], cfg.n[1], cfg.n[0], 3, 3)
    assert np.array_equal(s1, np.swapaxes(s1, -1, -2))
    # partition covers the grid exactly once
    cover = np.zeros(cfg.n[::-1], int)
    for (i0, i1, j0, j1, k0, k1) in cfg.boxes:
        cover[k0:k1, j0:j1, i0:i1] += 1
    assert np.all(cover == 1)
    # no source within 1e-6 h of a centroid (E0 singular there)
    cz, cy, cx = (cfg.cell_centers(2), cfg.cell_centers(1), cfg.cell_centers(0))
    for pos, _ in cfg.sources:
        d = np.sqrt((cx[None, None, :] - pos[0]) ** 2 + (cy[None, :, None] - pos[1]) ** 2 + (cz[:, None, None] - pos[2]) ** 2)
        assert d.min() > 1e-6 * cfg.h


def test_c1_recipe_literal():
    cfg = make_config("c1")
    s = cfg.sigma()
    ds = s - np.eye(3)
    inside = np.zeros((8, 8, 8), bool)
    inside[2:6, 2:6, 2:6] = True
    assert np.all(ds[~inside] == 0)
    d = ds[inside][:, 0, 0]
    assert d.min() >= 0.5 and d.max() <= 5.0
    assert np.all(ds[inside][:, 0, 1] == 0)


def test_c4_stations_inside_grid():
    st = c4_stations()
    assert len(st) == 64
    for s in st:
        for p in [s["tx"], *s["rx"]]:
            assert np.all(np.abs(p[:2]) <= 12.8) and abs(p[2]) <= 6.6
        F = s["moments"]
        assert np.abs(F @ F.T - np.eye(3)).max() < 1e-14


def test_box_grid_order():
    b = box_grid((8, 4, 2), (2, 2, 1))
    assert b[0] == (0, 4, 0, 2, 0, 2) and b[1] == (4, 8, 0, 2, 0, 2) and b[2] == (0, 4, 2, 4, 0, 2)


def test_logging_formation_and_window_rotation():
    """Formation tensors are symmetric positive definite; a window tensor is R^T sigma R of the
    formation at the mapped centroid (checked at one cell); sand cells are isotropic (Eq. 25)."""
    from ie_workloads import logging as lg
    n, h = (8, 4, 4), 1.0
    tx = lg.stations(4)[2]
    s = lg.window_sigma(tx, n, h, behind=3.0)
    assert np.abs(s - np.swapaxes(s, -1, -2)).max() < 1e-15
    assert np.linalg.eigvalsh(s).min() > 0
    origin, R = lg.window_grid(n, h, behind=3.0)
    i, j, k = 5, 1, 2
    r = tx + R @ (origin + h * np.array([i, j, k]))
    ref = R.T @ lg.formation_sigma(r[None])[0] @ R
    assert np.abs(s[k, j, i] - ref).max() < 1e-14
    assert abs(np.linalg.det(R) - 1) < 1e-14 and abs(R[:, 0] @ lg.hole_direction() - 1) < 1e-14
    # a sand point (Eq. 25): isotropic, perturbation peak at r_c
    z_sand = 0.5 * (lg.BEDS[5][0] + lg.BEDS[6][0]) + lg.bed_shift(500.0)
    sp = lg.formation_sigma(np.array([[500.0, 0.0, z_sand]]))[0]
    assert np.allclose(sp, sp[0, 0] * np.eye(3))
