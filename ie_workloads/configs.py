"""The BASELINE.json configurations c1..c5 as concrete synthetic inputs.

Grids are centred at the origin: origin_a = -(n_a - 1)/2 * h (centroid of cell (0,0,0)).
Seed = config number.  Readings for the parts BASELINE.json leaves open are listed in
DESIGN.md §Inputs; variants:
  c2capped  sigma_h ~ 10^U[-2,0] instead of 10^U[-2,1] (the literal c2
            contrast makes conventional-IE GMRES stagnate).  At 32^3 it still stagnates
            (oracle GMRES(30): relres 1.6e-4 after 3000 iterations; the resistive blocks,
            sigma_v down to 1e-3 S/m against sigma_b = 0.1, are the cause, not the cap)
  c2mod     the c2 geometry with moderate contrast: sigma_h = sigma_b 10^U[-0.3,0.7],
            sigma_v/sigma_h ~ U[0.3,1] (oracle GMRES(30) reaches 1e-11 in 56 iterations)
  c3, c4    the layered configs as BASELINE.json specifies them: three layers 1 / 0.01 / 1 S/m
            with interfaces at -4 / +4 m; tables and incident fields from layered_green (input data)
  c3capped  c3 with d_i <= min(5, 10 sigma_b(z))
  c3lmini, c4lmini  the c3 / c4 recipes on 8^3 with the interfaces scaled to -0.5 / +0.5 m
  c3h, c4h  the c3 / c4 grids, contrast recipes and tools on a HOMOGENEOUS background
            (c3h: sigma_b = 1 S/m; c4h: sigma_b = 0.01 S/m, the middle layer that holds the
            slab and the trajectory -- in a 1 S/m host the sigma_v = 0.005 slab is a 200x
            resistive body and conventional-IE GMRES stagnates at 3e-4); the layered path
            runs on the degenerate table (R19).
  *mini     the same recipe on an 8^3 grid so that dense LU gives exact truth.
"""

from dataclasses import dataclass, field
from typing import Callable, List, Tuple

import numpy as np

from .generate import vti_tensor, haar_rotation, gaussian_random_field, tool_frame, box_grid


@dataclass
class Config:
    name: str
    n: Tuple[int, int, int]          # (nx, ny, nz)
    h: float                         # cubic cell size, m
    sigma_b: float                   # background conductivity, S/m
    freq: float                      # Hz
    seed: int
    sigma_fn: Callable = None        # rng, cfg -> (nz, ny, nx, 3, 3) total sigma
    sources: List = field(default_factory=list)    # [(pos(3), moment(3))]
    receivers: List = field(default_factory=list)  # [pos(3)]
    boxes: List = field(default_factory=list)      # [(i0,i1,j0,j1,k0,k1)]
    restart: int = 30
    outer_tol: float = 1e-8
    parity_tol: float = 1e-9
    note: str = ""
    layers: Tuple = None             # layered background: sigma per layer, bottom -> top (S/m)
    z_iface: Tuple = None            # ascending interface depths (m); sigma_b is None then
    rx_moments: Tuple = None         # receiver dipole axes (rows); default x, y, z

    @property
    def layered(self):
        return self.layers is not None

    def background(self):
        """(sigma per layer, interfaces) -- a one-layer tuple for a homogeneous background."""
        if self.layered:
            return tuple(self.layers), tuple(self.z_iface)
        return (self.sigma_b,), ()

    def sigma_b_at(self, z):
        """Background conductivity at depth(s) z (layer l holds z_iface[l-1] <= z < z_iface[l])."""
        lay, zi = self.background()
        return np.asarray(lay, np.float64)[np.searchsorted(np.asarray(zi, np.float64), np.asarray(z, np.float64),
                                                          side="right")]

    @property
    def hvec(self):
        return (self.h, self.h, self.h)

    @property
    def origin(self):
        return tuple(-(na - 1) / 2.0 * self.h for na in self.n)

    @property
    def N(self):
        return self.n[0] * self.n[1] * self.n[2]

    def sigma(self):
        rng = np.random.default_rng(self.seed)
        return self.sigma_fn(rng, self)

    def cell_centers(self, axis):
        return self.origin[axis] + self.h * np.arange(self.n[axis])


# ---------------------------------------------------------------------------- recipes

def _c1_sigma(rng, cfg):
    """c1: central block [n/4, 3n/4)^3, isotropic Delta sigma ~ U[0.5, 5] per cell (x-fastest)."""
    nx, ny, nz = cfg.n
    s = np.zeros((nz, ny, nx, 3, 3))
    s[...] = cfg.sigma_b * np.eye(3)
    a, b = nx // 4, 3 * nx // 4
    d = rng.uniform(0.5, 5.0, size=(b - a, b - a, b - a))  # (z, y, x), x fastest
    s[a:b, a:b, a:b] += d[..., None, None] * np.eye(3)
    return s


def _blocks_vti(rng, cfg, block, log_hi):
    """c2: per block (x-fastest block order) draw sigma_h = 10^U[-2, log_hi], ratio U[0.1,1],
    dip U[0,60] deg, azimuth U[0,360] deg, in that order; Appendix C tensor."""
    nx, ny, nz = cfg.n
    s = np.zeros((nz, ny, nx, 3, 3))
    for kb in range(nz // block):
        for jb in range(ny // block):
            for ib in range(nx // block):
                sh = 10.0 ** rng.uniform(-2.0, log_hi)
                r = rng.uniform(0.1, 1.0)
                th = np.radians(rng.uniform(0.0, 60.0))
                ph = np.radians(rng.uniform(0.0, 360.0))
                s[kb * block:(kb + 1) * block, jb * block:(jb + 1) * block, ib * block:(ib + 1) * block] = \
                    vti_tensor(sh, r * sh, th, ph)
    return s


def _blocks_vti_mod(rng, cfg, block=8):
    """c2mod: per block (x-fastest) sigma_h = sigma_b 10^U[-0.3, 0.7], ratio U[0.3, 1], dip
    U[0,60] deg, azimuth U[0,360] deg, in that order; Appendix C tensor."""
    nx, ny, nz = cfg.n
    s = np.zeros((nz, ny, nx, 3, 3))
    for kb in range(nz // block):
        for jb in range(ny // block):
            for ib in range(nx // block):
                sh = cfg.sigma_b * 10.0 ** rng.uniform(-0.3, 0.7)
                r = rng.uniform(0.3, 1.0)
                th = np.radians(rng.uniform(0.0, 60.0))
                ph = np.radians(rng.uniform(0.0, 360.0))
                s[kb * block:(kb + 1) * block, jb * block:(jb + 1) * block, ib * block:(ib + 1) * block] = \
                    vti_tensor(sh, r * sh, th, ph)
    return s


def _c3_sigma(rng, cfg, block=16):
    """c3: one Haar rotation per block (x-fastest), then d_i = 10^U[-2, log10 5] per cell,
    shape (nz, ny, nx, 3); sigma = R diag(d) R^T."""
    nx, ny, nz = cfg.n
    nbx, nby, nbz = -(-nx // block), -(-ny // block), -(-nz // block)
    Rs = np.stack([haar_rotation(rng) for _ in range(nbx * nby * nbz)]).reshape(nbz, nby, nbx, 3, 3)
    d = 10.0 ** rng.uniform(-2.0, np.log10(5.0), size=(nz, ny, nx, 3))
    iz, iy, ix = np.meshgrid(np.arange(nz) // block, np.arange(ny) // block, np.arange(nx) // block, indexing="ij")
    R = Rs[iz, iy, ix]
    s = np.einsum("zyxij,zyxj,zyxkj->zyxik", R, d, R)
    return 0.5 * (s + np.swapaxes(s, -1, -2))  # exactly symmetric


def _c4_sigma(rng, cfg):
    """c4 (homogeneous stand-in): a 2 m slab through the origin with normal (sin30,0,cos30),
    TI sigma_h=0.02, sigma_v=0.005 about the normal (App. C, theta=30 deg, phi=0), in a
    sigma_b host; then 20 ellipsoids: centre U over the grid inset 2 m, semi-axes U[0.5,2] m,
    Haar rotation, eigenvalues sigma_b*10^U[-1,1]; later objects overwrite earlier ones."""
    nx, ny, nz = cfg.n
    s = np.zeros((nz, ny, nx, 3, 3))
    s[...] = cfg.sigma_b * np.eye(3)
    z, y, x = (cfg.cell_centers(2), cfg.cell_centers(1), cfg.cell_centers(0))
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    nrm = np.array([np.sin(np.radians(30)), 0.0, np.cos(np.radians(30))])
    dist = X * nrm[0] + Y * nrm[1] + Z * nrm[2]
    slab = np.abs(dist) <= 1.0
    s[slab] = vti_tensor(0.02, 0.005, np.radians(30.0), 0.0)
    lo = np.array([x[0], y[0], z[0]]) + 2.0
    hi = np.array([x[-1], y[-1], z[-1]]) - 2.0
    for _ in range(20):
        c = rng.uniform(lo, hi)
        ax = rng.uniform(0.5, 2.0, size=3)
        R = haar_rotation(rng)
        ev = cfg.sigma_b * 10.0 ** rng.uniform(-1.0, 1.0, size=3)
        P = np.stack([X - c[0], Y - c[1], Z - c[2]], axis=-1) @ R  # body-frame coordinates
        inside = np.sum((P / ax) ** 2, axis=-1) <= 1.0
        s[inside] = R @ np.diag(ev) @ R.T
    return s


def _c5_sigma(rng, cfg, corr_len=2.0, spread=0.3, block=10):
    """c5: three Gaussian random fields (correlation length 2 m); log10 d_i = log10 sigma_b +
    spread * z_i clipped to [-2, 1]; one Haar rotation per block^3 cells (x-fastest);
    sigma = R diag(d) R^T."""
    nx, ny, nz = cfg.n
    zf = [gaussian_random_field(rng, (nz, ny, nx), cfg.h, corr_len) for _ in range(3)]
    d = np.stack([10.0 ** np.clip(np.log10(cfg.sigma_b) + spread * f, -2.0, 1.0) for f in zf], axis=-1)
    nbx, nby, nbz = -(-nx // block), -(-ny // block), -(-nz // block)
    Rs = np.stack([haar_rotation(rng) for _ in range(nbx * nby * nbz)]).reshape(nbz, nby, nbx, 3, 3)
    iz, iy, ix = np.meshgrid(np.arange(nz) // block, np.arange(ny) // block, np.arange(nx) // block, indexing="ij")
    R = Rs[iz, iy, ix]
    s = np.einsum("zyxij,zyxj,zyxkj->zyxik", R, d, R)
    return 0.5 * (s + np.swapaxes(s, -1, -2))  # exactly symmetric


def _c3_sigma_capped(rng, cfg, block=16):
    """c3capped: as c3 but d_i = 10^(-2 + u (hi(z) + 2)), u ~ U[0,1] per cell
    (the same draws as c3), hi(z) = log10 min(5, 10 sigma_b(z)): contrast <= 9 sigma_b."""
    nx, ny, nz = cfg.n
    nbx, nby, nbz = -(-nx // block), -(-ny // block), -(-nz // block)
    Rs = np.stack([haar_rotation(rng) for _ in range(nbx * nby * nbz)]).reshape(nbz, nby, nbx, 3, 3)
    u = rng.uniform(0.0, 1.0, size=(nz, ny, nx, 3))
    hi = np.log10(np.minimum(5.0, 10.0 * cfg.sigma_b_at(cfg.cell_centers(2))))
    d = 10.0 ** (-2.0 + u * (hi[:, None, None, None] + 2.0))
    iz, iy, ix = np.meshgrid(np.arange(nz) // block, np.arange(ny) // block, np.arange(nx) // block, indexing="ij")
    R = Rs[iz, iy, ix]
    s = np.einsum("zyxij,zyxj,zyxkj->zyxik", R, d, R)
    return 0.5 * (s + np.swapaxes(s, -1, -2))


def _c4_sigma_layered(rng, cfg, slab_half=1.0, inset=2.0, n_ell=20, axes=(0.5, 2.0), slab_in_middle_only=False):
    """c4 (layered, BASELINE.json configs[3]): background sigma_b(z) of the three layers, then a
    slab of half-thickness 1 m through the origin with normal (sin30, 0, cos30), TI sigma_h = 0.02,
    sigma_v = 0.005 about the normal (App. C, theta = 30 deg, phi = 0); then 20 ellipsoids:
    centre U over the grid inset 2 m, semi-axes U[0.5, 2] m, Haar rotation R, eigenvalue RATIOS
    r = 10^U[-1, 1]; an ellipsoid cell takes sigma_b(z_cell) R diag(r) R^T, i.e. its contrast
    to the local background stays in [-0.9, 9] even where it crosses an interface (DESIGN.md
    R22; BASELINE.json leaves the inclusions' values open); later objects overwrite earlier ones."""
    nx, ny, nz = cfg.n
    z, y, x = (cfg.cell_centers(2), cfg.cell_centers(1), cfg.cell_centers(0))
    s = np.zeros((nz, ny, nx, 3, 3))
    s[...] = cfg.sigma_b_at(z)[:, None, None, None, None] * np.eye(3)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    nrm = np.array([np.sin(np.radians(30)), 0.0, np.cos(np.radians(30))])
    slab = np.abs(X * nrm[0] + Y * nrm[1] + Z * nrm[2]) <= slab_half
    if slab_in_middle_only:  # c4mid: the slab ends at the interfaces (a bed of the middle layer)
        slab &= cfg.sigma_b_at(Z) == min(cfg.layers)
    s[slab] = vti_tensor(0.02, 0.005, np.radians(30.0), 0.0)
    lo = np.array([x[0], y[0], z[0]]) + inset
    hi = np.array([x[-1], y[-1], z[-1]]) - inset
    for _ in range(n_ell):
        c = rng.uniform(lo, hi)
        ax = rng.uniform(axes[0], axes[1], size=3)
        R = haar_rotation(rng)
        ratio = 10.0 ** rng.uniform(-1.0, 1.0, size=3)
        P = np.stack([X - c[0], Y - c[1], Z - c[2]], axis=-1) @ R
        inside = np.sum((P / ax) ** 2, axis=-1) <= 1.0
        s[inside] = cfg.sigma_b_at(Z[inside])[:, None, None] * (R @ np.diag(ratio) @ R.T)
    return s


# ------------------------------------------------------------------------- c4 stations

def c4_stations(n_stations=64, incl=70.0, azim=45.0, spacings=(1.0, 3.0, 7.0)):
    """Trajectory through the origin, inclination 70 deg, azimuth 45 deg; station s at
    t_s = -3.5 + (s - 31.5) * 0.5 m along d; receivers at Tx + {1,3,7} d; triaxial dipoles
    along the tool axes x', y', z'.  Returns list of dict(tx, moments(3x3), rx(3x3))."""
    F = tool_frame(incl, azim)
    d = F[2]
    out = []
    for s in range(n_stations):
        t = -3.5 + (s - 31.5) * 0.5
        tx = t * d
        out.append(dict(tx=tx, moments=F.copy(), rx=np.stack([tx + L * d for L in spacings])))
    return out


# ---------------------------------------------------------------------------- registry

def make_config(name):
    zdip = np.array([0.0, 0.0, 1.0])
    tri = np.eye(3)
    if name == "c1":
        return Config("c1", (8, 8, 8), 0.25, 1.0, 1e5, 1, _c1_sigma,
                      sources=[(np.array([0.0, 0.0, 1.0]), zdip)], receivers=[np.array([0.0, 0.0, 2.0])],
                      boxes=[(0, 8, 0, 8, 0, 8)], restart=30, outer_tol=1e-10, parity_tol=1e-10)
    if name in ("c2", "c2capped"):
        log_hi = 1.0 if name == "c2" else 0.0
        return Config(name, (32, 32, 32), 0.1, 0.1, 2e6, 2, lambda rng, c: _blocks_vti(rng, c, 8, log_hi),
                      sources=[(np.zeros(3), zdip)],
                      receivers=[np.array([0.0, 0.0, 0.5]), np.array([0.0, 0.0, 1.0])],
                      boxes=[(0, 32, 0, 32, 0, 16), (0, 32, 0, 32, 16, 32)], restart=30, outer_tol=1e-8)
    if name == "c2mod":
        return Config(name, (32, 32, 32), 0.1, 0.1, 2e6, 2, _blocks_vti_mod,
                      sources=[(np.zeros(3), zdip)],
                      receivers=[np.array([0.0, 0.0, 0.5]), np.array([0.0, 0.0, 1.0])],
                      boxes=[(0, 32, 0, 32, 0, 16), (0, 32, 0, 32, 16, 32)], restart=30, outer_tol=1e-8)
    if name == "c2mini":
        return Config(name, (8, 8, 8), 0.1, 0.1, 2e6, 2, lambda rng, c: _blocks_vti(rng, c, 2, 0.0),
                      sources=[(np.zeros(3), zdip)], receivers=[np.array([0.0, 0.0, 0.5])],
                      boxes=[(0, 8, 0, 8, 0, 4), (0, 8, 0, 8, 4, 8)], restart=30, outer_tol=1e-9)
    if name == "c3h":
        return Config(name, (64, 64, 64), 0.25, 1.0, 4e5, 3, _c3_sigma,
                      sources=[(np.zeros(3), tri[i]) for i in range(3)],
                      receivers=[np.array([0.0, 0.0, z]) for z in (1.0, 3.0, 7.0)],
                      boxes=box_grid((64, 64, 64), (2, 2, 1)), restart=30, outer_tol=1e-8,
                      note="homogeneous stand-in for the layered c3 (sigma_b = 1 S/m)")
    if name == "c3mini":
        return Config(name, (8, 8, 8), 0.25, 1.0, 4e5, 3, lambda rng, c: _c3_sigma(rng, c, 4),
                      sources=[(np.zeros(3), tri[i]) for i in range(3)],
                      receivers=[np.array([0.0, 0.0, 1.0])],
                      boxes=box_grid((8, 8, 8), (2, 2, 1)), restart=30, outer_tol=1e-9)
    if name == "c4h":
        st = c4_stations()
        return Config(name, (128, 128, 64), 0.25, 0.01, 4e5, 4, _c4_sigma,
                      sources=[(st[31]["tx"], st[31]["moments"][i]) for i in range(3)],
                      receivers=list(st[31]["rx"]),
                      boxes=box_grid((128, 128, 64), (4, 2, 1)), restart=30, outer_tol=1e-6,
                      note="homogeneous stand-in for the layered c4 at its middle-layer conductivity "
                           "(sigma_b = 0.01 S/m, 400 kHz): the slab and the trajectory sit in that layer")
    lay3 = dict(layers=(1.0, 0.01, 1.0), z_iface=(-4.0, 4.0))
    lay3mini = dict(layers=(1.0, 0.01, 1.0), z_iface=(-0.5, 0.5))
    if name in ("c3", "c3capped"):
        return Config(name, (64, 64, 64), 0.25, None, 4e5, 3, _c3_sigma if name == "c3" else _c3_sigma_capped,
                      sources=[(np.zeros(3), tri[i]) for i in range(3)],
                      receivers=[np.array([0.0, 0.0, z]) for z in (1.0, 3.0, 7.0)],
                      boxes=box_grid((64, 64, 64), (2, 2, 1)), restart=30, outer_tol=1e-8, **lay3,
                      note="three-layer background 1 / 0.01 / 1 S/m, interfaces at -4 / +4 m (physical table)")
    if name in ("c3lmini", "c3lminicapped"):
        fn = (lambda rng, c: _c3_sigma(rng, c, 4)) if name == "c3lmini" else (lambda rng, c: _c3_sigma_capped(rng, c, 4))
        return Config(name, (8, 8, 8), 0.25, None, 4e5, 3, fn,
                      sources=[(np.zeros(3), tri[i]) for i in range(3)],
                      receivers=[np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, -1.5])],
                      boxes=box_grid((8, 8, 8), (2, 2, 1)), restart=30, outer_tol=1e-9, **lay3mini,
                      note="c3 recipe on 8^3 with the interfaces scaled to -0.5 / +0.5 m")
    if name == "c4":
        st = c4_stations()
        return Config(name, (128, 128, 64), 0.25, None, 4e5, 4, _c4_sigma_layered,
                      sources=[(st[31]["tx"], st[31]["moments"][i]) for i in range(3)],
                      receivers=list(st[31]["rx"]), rx_moments=tuple(map(tuple, st[31]["moments"])),
                      boxes=box_grid((128, 128, 64), (4, 2, 1)), restart=30, outer_tol=1e-6, **lay3,
                      note="three-layer background 1 / 0.01 / 1 S/m (physical table); station 31 of the sweep")
    if name == "c4mid":
        st = c4_stations()
        return Config(name, (128, 128, 64), 0.25, None, 4e5, 4,
                      lambda rng, c: _c4_sigma_layered(rng, c, slab_in_middle_only=True),
                      sources=[(st[31]["tx"], st[31]["moments"][i]) for i in range(3)],
                      receivers=list(st[31]["rx"]), rx_moments=tuple(map(tuple, st[31]["moments"])),
                      boxes=box_grid((128, 128, 64), (4, 2, 1)), restart=30, outer_tol=1e-6, **lay3,
                      note="c4 with the resistive slab confined to the middle layer (in the 1 S/m shoulders "
                           "it is a 200x resistive sheet that stalls the DD iterations)")
    if name == "c4lmini":
        F = tool_frame(70.0, 45.0)
        tx = 0.1 * F[2]
        return Config(name, (8, 8, 8), 0.25, None, 4e5, 4,
                      lambda rng, c: _c4_sigma_layered(rng, c, slab_half=0.25, inset=0.5, n_ell=3, axes=(0.25, 0.5)),
                      sources=[(tx, F[i]) for i in range(3)], receivers=[tx + 0.6 * F[2], tx + 1.2 * F[2]],
                      rx_moments=tuple(map(tuple, F)), boxes=box_grid((8, 8, 8), (2, 2, 1)), restart=30,
                      outer_tol=1e-9, **lay3mini, note="c4 recipe scaled to 8^3 (interfaces at -0.5 / +0.5 m)")
    if name == "c5":
        return Config(name, (256, 256, 128), 0.2, 0.5, 1e5, 5, _c5_sigma,
                      sources=[(np.zeros(3), zdip)],
                      receivers=[np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, 3.0])],
                      boxes=box_grid((256, 256, 128), (4, 4, 1)), restart=50, outer_tol=1e-6)
    if name == "c5jac":
        return Config(name, (128, 128, 128), 0.2, 0.5, 1e5, 5, _c5_sigma,
                      sources=[(np.zeros(3), zdip)], receivers=[np.array([0.0, 0.0, 1.0])],
                      boxes=box_grid((128, 128, 128), (2, 2, 1)), restart=50, outer_tol=1e-6,
                      note="the c5 recipe on 128^3 with 2x2 boxes of 64x64x128 (the c5 box shape): the "
                           "oracle's block Jacobi runs here sweep by sweep beside the GPU's")
    if name == "c5mini":
        return Config(name, (8, 8, 8), 0.2, 0.5, 1e5, 5, lambda rng, c: _c5_sigma(rng, c, corr_len=0.4, block=2),
                      sources=[(np.zeros(3), zdip)], receivers=[np.array([0.0, 0.0, 1.0])],
                      boxes=box_grid((8, 8, 8), (2, 2, 1)), restart=50, outer_tol=1e-9)
    raise KeyError(name)


CONFIG_NAMES = ("c1", "c2", "c2capped", "c2mod", "c2mini", "c3h", "c3mini", "c4h", "c5", "c5mini",
                "c3", "c3capped", "c3lmini", "c3lminicapped", "c4", "c4mid", "c4lmini", "c5jac")
