"""The paper's logging workload (section 3.3) as synthetic inputs: a faulted,
gently dipping shale/sand formation, an 85-degree trajectory from (0,0,0) to (900,0,78.74) m,
and the moving forward-modelling window aligned with the drilling direction.

Inputs only (no arithmetic of the IE method): the formation is an analytic function of position,
a window is sampled at its cell centroids in global coordinates and the tensors are expressed in
the window frame (the rotation of Appendix C, written as R^T sigma R).  The paper's
geometry exists only in its figures; the recipe below has its stated ingredients:
  * anisotropic (TI) shale layers around isotropic sand layers, 2.5-D (invariant along y),
    beds dipping DIP_DEG along x, a normal fault at x = FAULT_X throwing the beds by FAULT_THROW;
  * the sand perturbation of Eq. 25: sigma = sigma_u (1 + alpha exp(-|r - r_c| / gamma)),
    r_c = (500, 0, 40) m, alpha = 4, gamma = 50 m;
  * tool: transmitter along the hole axis, 24 kHz, receivers 7, 15, 30 m ahead;
  * window background sigma0 = 0.1 S/m, cell 0.25 m.
The window's long axis is its x axis (the hole direction) -- the paper points its z axis there;
the physics is the same and the FFT lengths map onto the fast kernels.
"""

import numpy as np

DIP_DEG = 2.0
FAULT_X, FAULT_THROW = 620.0, 12.0
# bed tops (m, at x = 0, before dip and fault) from the top down: (top, kind, sigma_h, sigma_v|sigma_u)
BEDS = [(+1e9, "shale", 0.4, 0.1),
        (95.0, "sand", 0.05, None),
        (70.0, "shale", 0.3, 0.075),
        (52.0, "sand", 0.04, None),
        (30.0, "shale", 0.5, 0.125),
        (12.0, "sand", 0.06, None),
        (-6.0, "shale", 0.4, 0.1)]  # shale 2-3.3 ohm-m horizontal, anisotropy ratio 4
R_C, ALPHA, GAMMA = np.array([500.0, 0.0, 40.0]), 4.0, 50.0
START, END = np.array([0.0, 0.0, 0.0]), np.array([900.0, 0.0, 78.74])
FREQ, SIGMA0, SPACINGS = 24e3, 0.1, (7.0, 15.0, 30.0)


def bed_shift(x):
    """Vertical displacement of the beds at x: dip plus the fault throw beyond FAULT_X."""
    return x * np.tan(np.radians(DIP_DEG)) + np.where(x > FAULT_X, -FAULT_THROW, 0.0)


def formation_sigma(r):
    """Total conductivity tensor (..., 3, 3) at global points r (..., 3)."""
    r = np.asarray(r, np.float64)
    x, z = r[..., 0], r[..., 2]
    zr = z - bed_shift(x)  # depth in the undisturbed bed frame
    out = np.zeros(r.shape[:-1] + (3, 3))
    # symmetry axis of the TI shale: the bed normal, tilted by the dip about y
    d = np.radians(DIP_DEG)
    n = np.array([-np.sin(d), 0.0, np.cos(d)])
    nn = np.outer(n, n)
    pert = 1.0 + ALPHA * np.exp(-np.linalg.norm(r - R_C, axis=-1) / GAMMA)
    for i, (top, kind, a, b) in enumerate(BEDS):
        bottom = BEDS[i + 1][0] if i + 1 < len(BEDS) else -1e9
        m = (zr < top) & (zr >= bottom)
        if kind == "shale":
            out[m] = a * np.eye(3) + (b - a) * nn
        else:
            out[m] = (a * pert[m])[:, None, None] * np.eye(3)
    return out


def hole_direction():
    v = END - START
    return v / np.linalg.norm(v)


def window_frame():
    """Rotation R (columns = the window's x, y, z axes in global coordinates): x along the
    hole, y horizontal (global y), z = x cross y."""
    ex = hole_direction()
    ey = np.array([0.0, 1.0, 0.0])
    ez = np.cross(ex, ey)
    return np.stack([ex, ey, ez], axis=1)


def stations(n):
    """n transmitter positions evenly spaced along the trajectory."""
    t = np.linspace(0.0, 1.0, n)
    return START[None, :] + t[:, None] * (END - START)[None, :]


def window_grid(n, h, behind=17.0):
    """Window of n = (nx, ny, nz) cells of size h in its own frame: the transmitter sits on the
    window axis, `behind` metres from the trailing face, so receivers up to ~n_x h - behind
    ahead fit.  Returns (origin of cell (0,0,0) relative to the transmitter, window frame)."""
    nx, ny, nz = n
    origin = np.array([-behind + h / 2, -(ny - 1) / 2 * h, -(nz - 1) / 2 * h])
    return origin, window_frame()


def window_sigma(tx, n, h, behind=17.0):
    """Conductivity of the window at station tx, in the window frame: sigma' = R^T sigma(r) R at
    the centroids r = tx + R (origin + (i, j, k) h).  Returns (nz, ny, nx, 3, 3)."""
    origin, R = window_grid(n, h, behind)
    nx, ny, nz = n
    z, y, x = np.meshgrid(origin[2] + h * np.arange(nz), origin[1] + h * np.arange(ny),
                          origin[0] + h * np.arange(nx), indexing="ij")
    local = np.stack([x, y, z], axis=-1)
    glob = tx + local @ R.T
    s = formation_sigma(glob)
    return np.einsum("ia,...ij,jb->...ab", R, s, R)


def tool_in_window():
    """Transmitter at the window origin of the tool frame (0,0,0), moment along the hole axis
    (the window x axis); receivers ahead on the axis."""
    return (np.zeros(3), np.array([1.0, 0.0, 0.0]), [np.array([s, 0.0, 0.0]) for s in SPACINGS])


def window_sigma_device(tx, n, h, behind=17.0, device="cuda"):
    """window_sigma evaluated with torch on the device (the formation is an analytic function of
    position, so a station's window needs no host work or H2D copy): the same recipe, the same
    float64 arithmetic, returned as a (nz, ny, nx, 3, 3) float64 tensor on `device`.  Input
    generation only (torch elementwise ops), like the numpy version."""
    import torch
    origin, R = window_grid(n, h, behind)
    nx, ny, nz = n
    f64 = dict(dtype=torch.float64, device=device)
    Rt = torch.tensor(R, **f64)
    z = origin[2] + h * torch.arange(nz, **f64)
    y = origin[1] + h * torch.arange(ny, **f64)
    x = origin[0] + h * torch.arange(nx, **f64)
    Z, Y, X = torch.meshgrid(z, y, x, indexing="ij")
    local = torch.stack([X, Y, Z], dim=-1)
    glob = torch.tensor(np.asarray(tx, np.float64), **f64) + local @ Rt.T
    gx, gz = glob[..., 0], glob[..., 2]
    shift = gx * np.tan(np.radians(DIP_DEG)) + torch.where(gx > FAULT_X, -FAULT_THROW, 0.0)
    zr = gz - shift
    d = np.radians(DIP_DEG)
    nvec = torch.tensor([-np.sin(d), 0.0, np.cos(d)], **f64)
    nn = torch.outer(nvec, nvec)
    eye = torch.eye(3, **f64)
    pert = 1.0 + ALPHA * torch.exp(-torch.linalg.vector_norm(glob - torch.tensor(R_C, **f64), dim=-1) / GAMMA)
    s = torch.zeros(glob.shape[:-1] + (3, 3), **f64)
    for i, (top, kind, a, b) in enumerate(BEDS):
        bottom = BEDS[i + 1][0] if i + 1 < len(BEDS) else -1e9
        m = ((zr < top) & (zr >= bottom))[..., None, None]
        if kind == "shale":
            val = (a * eye + (b - a) * nn).expand_as(s)
        else:
            val = (a * pert)[..., None, None] * eye
        s = torch.where(m, val, s)
    return torch.einsum("ia,...ij,jb->...ab", Rt, s, Rt).contiguous()
