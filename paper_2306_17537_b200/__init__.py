"""Thin ctypes binding of libie_b200.so (include/ie_b200.h).

Argument marshalling only: every step of the method runs in the CUDA library.  torch is used
for device memory (tensors' data pointers) and streams.  There is NO CPU fallback: importing
works without a GPU (so the symbol table can be checked), but every call that needs the
device fails loudly if the library or the GPU is missing.

Function names follow the C-ABI (ie_create, ie_set_contrast, ie_set_source, ie_apply_operator,
ie_solve_subdomain, ie_solve_dd, ie_receiver_fields, ...).
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IE_LIB_PATH") or os.path.join(HERE, "libie_b200.so")  # IE_LIB_PATH: A/B of an alternative build (tools/gpu_ab_lib.sh)

IE_OK = 0
STATUS = {0: "IE_OK", 1: "IE_ERR_INVALID_ARGUMENT", 2: "IE_ERR_OUT_OF_MEMORY", 3: "IE_ERR_CUDA",
          4: "IE_ERR_NOT_CONVERGED", 5: "IE_ERR_BREAKDOWN", 6: "IE_ERR_STATE", 7: "IE_ERR_PLACEMENT",
          8: "IE_ERR_UNSUPPORTED"}
IE_DD_FULL, IE_DD_JACOBI, IE_DD_GAUSS_SEIDEL, IE_DD_FGMRES_JACOBI, IE_DD_FGMRES_GAUSS_SEIDEL = 0, 1, 2, 3, 4
SCHEMES = {"full": IE_DD_FULL, "jacobi": IE_DD_JACOBI, "gauss_seidel": IE_DD_GAUSS_SEIDEL,
           "fgmres_jacobi": IE_DD_FGMRES_JACOBI, "fgmres_gauss_seidel": IE_DD_FGMRES_GAUSS_SEIDEL}

EXPORTED = ("ie_create", "ie_destroy", "ie_last_error", "ie_workspace_query", "ie_bind_workspace",
            "ie_set_contrast", "ie_set_source", "ie_get_incident", "ie_set_incident", "ie_apply_operator",
            "ie_solve_subdomain", "ie_solve_dd", "ie_solve_dd_warm", "ie_set_preconditioner", "ie_receiver_fields",
            "ie_get_info", "ie_get_green_octant",
            "ie_profile", "ie_profile_read", "ie_receiver_fields_table", "ie_get_layer_spectrum")
IE_TABLE_NONE, IE_TABLE_QUADRANT, IE_TABLE_HOMOGENEOUS = 0, 1, 2
KERNELS = ("K-A x-forward+contrast", "K-B y-forward", "K-C z-convolution", "K-D y-inverse",
           "K-E x-inverse+update", "K-DE y-inverse+x-inverse+update (fused)",
           "K-AB contrast+x-forward+y-forward (fused)")


class IEError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ie_grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
                ("origin", ctypes.c_double * 3)]


class ie_background(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("sigma", ctypes.POINTER(ctypes.c_double)),
                ("z_iface", ctypes.POINTER(ctypes.c_double)), ("table", ctypes.c_void_p),
                ("table_format", ctypes.c_int32)]


class ie_box(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("i0", "i1", "j0", "j1", "k0", "k1")]


class ie_gmres_opts(ctypes.Structure):
    _fields_ = [("restart", ctypes.c_int32), ("max_iters", ctypes.c_int32), ("min_iters", ctypes.c_int32),
                ("tol", ctypes.c_double)]


class ie_solve_stats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("restarts", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("relres_est", ctypes.c_double), ("relres_true", ctypes.c_double)]


class ie_dd_opts(ctypes.Structure):
    _fields_ = [("scheme", ctypes.c_int32), ("boxes", ctypes.POINTER(ie_box)), ("n_boxes", ctypes.c_int32),
                ("outer_tol", ctypes.c_double), ("adaptive", ctypes.c_int32), ("inner_tol_fixed", ctypes.c_double),
                ("inner_tol_factor", ctypes.c_double), ("max_sweeps", ctypes.c_int32), ("inner", ie_gmres_opts)]


class ie_dd_stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int32), ("total_inner_iters", ctypes.c_int32), ("full_applies", ctypes.c_int32),
                ("sub_applies", ctypes.c_int32), ("e_final", ctypes.c_double),
                ("e_hist", ctypes.POINTER(ctypes.c_double)), ("iters", ctypes.POINTER(ctypes.c_int32))]


class ie_info(ctypes.Structure):
    _fields_ = [("k0_re", ctypes.c_double), ("k0_im", ctypes.c_double), ("self_re", ctypes.c_double),
                ("self_im", ctypes.c_double), ("n_src", ctypes.c_int32), ("kernel_launches", ctypes.c_int32)]


_lib = None


def load_library(path=LIB_PATH):
    """Load libie_b200.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I, D, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_size_t
    sig = {
        "ie_create": [ctypes.POINTER(ie_grid), ctypes.POINTER(ie_background), D, P, ctypes.POINTER(P)],
        "ie_destroy": [P],
        "ie_workspace_query": [P, ctypes.POINTER(ie_box), I, I, I, ctypes.POINTER(S)],
        "ie_bind_workspace": [P, P, S],
        "ie_set_contrast": [P, P, I],
        "ie_set_source": [P, I, P, P],
        "ie_get_incident": [P, P],
        "ie_set_incident": [P, I, P],
        "ie_apply_operator": [P, ctypes.POINTER(ie_box), I, P, P],
        "ie_solve_subdomain": [P, ctypes.POINTER(ie_box), I, P, P, ctypes.POINTER(ie_gmres_opts),
                               ctypes.POINTER(ie_solve_stats)],
        "ie_solve_dd": [P, ctypes.POINTER(ie_dd_opts), P, ctypes.POINTER(ie_dd_stats)],
        "ie_solve_dd_warm": [P, ctypes.POINTER(ie_dd_opts), P, ctypes.POINTER(ie_dd_stats)],
        "ie_set_preconditioner": [P, I],
        "ie_receiver_fields": [P, P, I, P, P, P],
        "ie_get_info": [P, ctypes.POINTER(ie_info)],
        "ie_get_green_octant": [P, ctypes.POINTER(ie_box), P],
        "ie_profile": [P, I],
        "ie_profile_read": [P, P, P],
        "ie_receiver_fields_table": [P, P, I, P, P, P],
        "ie_get_layer_spectrum": [P, ctypes.POINTER(ie_box), P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.ie_last_error.argtypes = [P]
    lib.ie_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _ptr(t):
    """Device (or host) pointer of a torch tensor / numpy array; None -> NULL."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        assert t.is_contiguous(), "tensors must be contiguous"
        return ctypes.c_void_p(t.data_ptr())
    assert t.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(t.ctypes.data)


def _box(b):
    if b is None:
        return None
    return ctypes.byref(ie_box(*[int(v) for v in b]))


class IECtx:
    """Opaque context handle (ie_ctx*) plus the workspace tensor that is bound to it."""

    def __init__(self, handle, grid):
        self.handle = handle
        self.grid = grid
        self.workspace = None
        self.n_src = 0

    def last_error(self):
        msg = _lib.ie_last_error(self.handle) if _lib is not None else None
        return msg.decode() if msg else ""

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.ie_destroy(self.handle)
        except Exception:
            pass
        self.handle = None


def _check(ctx, st, what):
    if st != IE_OK:
        msg = _lib.ie_last_error(ctx.handle if ctx is not None else None)
        raise IEError(st, f"{what}: {msg.decode() if msg else ''}")


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def ie_create(n, h, origin, sigma_b, freq_hz, stream=None, table=None, table_format=None, z_iface=None):
    """n = (nx, ny, nz); h = (dx, dy, dz) m; origin = centroid of cell (0,0,0).

    Homogeneous background: sigma_b a number.  Layered (include/ie_b200.h): sigma_b a list of
    layer conductivities (bottom to top) with z_iface, and table = host complex128 numpy array
    [9][nz][nz][ny][nx] (format 1); or table_format=2 (the library's degenerate table)."""
    lib = load_library()
    g = ie_grid(int(n[0]), int(n[1]), int(n[2]), float(h[0]), float(h[1]), float(h[2]),
                (ctypes.c_double * 3)(*[float(v) for v in origin]))
    layers = np.atleast_1d(np.asarray(sigma_b, np.float64))
    sig = (ctypes.c_double * len(layers))(*layers)
    zi = None
    if z_iface is not None and len(z_iface):
        zi = (ctypes.c_double * len(z_iface))(*[float(v) for v in z_iface])
    fmt = table_format if table_format is not None else (IE_TABLE_QUADRANT if table is not None else IE_TABLE_NONE)
    tab = None
    if table is not None:
        table = np.ascontiguousarray(table, np.complex128)
        nx, ny, nz = (int(v) for v in n)
        assert table.size == 9 * nz * nz * ny * nx, "table must be [9][nz][nz][ny][nx]"
        tab = ctypes.c_void_p(table.ctypes.data)
    bg = ie_background(len(layers), sig, zi, tab, int(fmt))
    out = ctypes.c_void_p()
    st = lib.ie_create(ctypes.byref(g), ctypes.byref(bg), float(freq_hz), _stream_ptr(stream), ctypes.byref(out))
    if st != IE_OK:
        raise IEError(st, "ie_create: " + (lib.ie_last_error(None) or b"").decode())
    return IECtx(out, g)


def ie_workspace_query(ctx, boxes=None, nrhs=1, restart=30):
    bx = None
    nb = 0
    if boxes:
        arr = (ie_box * len(boxes))(*[ie_box(*[int(v) for v in b]) for b in boxes])
        bx, nb = arr, len(boxes)
    out = ctypes.c_size_t()
    _check(ctx, _lib.ie_workspace_query(ctx.handle, bx, nb, int(nrhs), int(restart), ctypes.byref(out)),
           "ie_workspace_query")
    return out.value


def ie_bind_workspace(ctx, ws):
    """ws: a CUDA uint8 tensor (kept alive by the context handle)."""
    ctx.workspace = ws
    _check(ctx, _lib.ie_bind_workspace(ctx.handle, _ptr(ws), ws.numel() * ws.element_size()), "ie_bind_workspace")


def ensure_workspace(ctx, boxes=None, nrhs=1, restart=30):
    """Query, allocate (torch, on the current device) and bind the scratch workspace."""
    import torch
    need = ie_workspace_query(ctx, boxes, nrhs, restart)
    if ctx.workspace is None or ctx.workspace.numel() < need:
        ctx.workspace = None
        ws = torch.empty(need + 256, dtype=torch.uint8, device="cuda")
        off = (-ws.data_ptr()) % 256
        ie_bind_workspace(ctx, ws[off:off + need])
        ctx.workspace_base = ws
    return need


def ie_set_contrast(ctx, sigma, layout=0):
    """sigma: CUDA float64 tensor (nz, ny, nx, 3, 3) (layout 0) or (6, nz, ny, nx) (layout 1), total sigma."""
    _check(ctx, _lib.ie_set_contrast(ctx.handle, _ptr(sigma), int(layout)), "ie_set_contrast")


def ie_set_source(ctx, pos, moment):
    pos = np.ascontiguousarray(np.asarray(pos, np.float64).reshape(-1, 3))
    mom = np.ascontiguousarray(np.asarray(moment, np.float64).reshape(-1, 3))
    assert pos.shape == mom.shape
    _check(ctx, _lib.ie_set_source(ctx.handle, len(pos), _ptr(pos), _ptr(mom)), "ie_set_source")
    ctx.n_src = len(pos)


def ie_get_incident(ctx, out):
    _check(ctx, _lib.ie_get_incident(ctx.handle, _ptr(out)), "ie_get_incident")


def ie_set_incident(ctx, e0):
    _check(ctx, _lib.ie_set_incident(ctx.handle, int(e0.shape[0]), _ptr(e0)), "ie_set_incident")
    ctx.n_src = int(e0.shape[0])


def ie_apply_operator(ctx, x, y, box=None):
    """y = (I - G dsigma) x on the grid or a box; x, y complex128 CUDA tensors [nrhs][3][bz][by][bx]."""
    nrhs = x.shape[0] if x.dim() == 5 else 1
    _check(ctx, _lib.ie_apply_operator(ctx.handle, _box(box), int(nrhs), _ptr(x), _ptr(y)), "ie_apply_operator")


def ie_set_preconditioner(ctx, kind):
    """0: conventional IE (the paper's); 1: contraction-IE right preconditioner, for every later solve."""
    _check(ctx, _lib.ie_set_preconditioner(ctx.handle, int(kind)), "ie_set_preconditioner")


def ie_solve_subdomain(ctx, b, x, tol, restart=30, max_iters=5000, min_iters=0, box=None, check=True, precond=0):
    nrhs = b.shape[0] if b.dim() == 5 else 1
    ie_set_preconditioner(ctx, precond)
    o = ie_gmres_opts(int(restart), int(max_iters), int(min_iters), float(tol))
    st = (ie_solve_stats * nrhs)()
    s = _lib.ie_solve_subdomain(ctx.handle, _box(box), int(nrhs), _ptr(b), _ptr(x), ctypes.byref(o), st)
    stats = [dict(iters=t.iters, restarts=t.restarts, converged=bool(t.converged), relres_est=t.relres_est,
                  relres_true=t.relres_true) for t in st]
    if check:
        _check(ctx, s, "ie_solve_subdomain")
    return stats, s


def ie_solve_dd(ctx, e, scheme, boxes=(), outer_tol=1e-8, adaptive=True, inner_tol_fixed=1e-6,
                inner_tol_factor=0.1, max_sweeps=200, restart=30, max_iters=2000, min_iters=1,
                init_from_e=False, check=True, precond=0):
    """Algorithm 1 (or full-domain GMRES for scheme="full").  e: [n_src][3][nz][ny][nx] CUDA tensor."""
    ns = ctx.n_src
    nb = len(boxes)
    arr = (ie_box * max(nb, 1))(*[ie_box(*[int(v) for v in b]) for b in boxes])
    o = ie_dd_opts(SCHEMES[scheme] if isinstance(scheme, str) else int(scheme), arr, nb, float(outer_tol),
                   int(bool(adaptive)), float(inner_tol_fixed), float(inner_tol_factor), int(max_sweeps),
                   ie_gmres_opts(int(restart), int(max_iters), int(min_iters), 0.0))
    ie_set_preconditioner(ctx, precond)
    e_hist = np.zeros(((max_sweeps + 1), ns), np.float64)
    iters = np.zeros((max(max_sweeps, 1), max(nb, 1), ns), np.int32)
    st = ie_dd_stats(0, 0, 0, 0, 0.0, e_hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     iters.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    fn = _lib.ie_solve_dd_warm if init_from_e else _lib.ie_solve_dd
    s = fn(ctx.handle, ctypes.byref(o), _ptr(e), ctypes.byref(st))
    out = dict(sweeps=st.sweeps, total_inner_iters=st.total_inner_iters, full_applies=st.full_applies,
               sub_applies=st.sub_applies, e_final=st.e_final, e_hist=e_hist[:st.sweeps + 1].copy(),
               iters=iters[:st.sweeps].copy(), status=s)
    if check:
        _check(ctx, s, "ie_solve_dd")
    return out


def ie_receiver_fields(ctx, e, rx):
    """Returns (H [n_src][n_rx][3], V [n_src][n_rx][3]) complex128 numpy arrays."""
    rx = np.ascontiguousarray(np.asarray(rx, np.float64).reshape(-1, 3))
    H = np.zeros((ctx.n_src, len(rx), 3), np.complex128)
    V = np.zeros_like(H)
    _check(ctx, _lib.ie_receiver_fields(ctx.handle, _ptr(e), len(rx), _ptr(rx), _ptr(H), _ptr(V)),
           "ie_receiver_fields")
    return H, V


def ie_get_info(ctx):
    inf = ie_info()
    _check(ctx, _lib.ie_get_info(ctx.handle, ctypes.byref(inf)), "ie_get_info")
    return dict(k0=complex(inf.k0_re, inf.k0_im), self_term=complex(inf.self_re, inf.self_im), n_src=inf.n_src,
                kernel_launches=inf.kernel_launches)


def ie_get_green_octant(ctx, box=None):
    if box is None:
        nx, ny, nz = ctx.grid.nx, ctx.grid.ny, ctx.grid.nz
    else:
        nx, ny, nz = box[1] - box[0], box[3] - box[2], box[5] - box[4]
    out = np.zeros((6, nz + 1, ny + 1, nx + 1), np.complex128)
    _check(ctx, _lib.ie_get_green_octant(ctx.handle, _box(box), _ptr(out)), "ie_get_green_octant")
    return out


def ie_profile(ctx, enable=True):
    _check(ctx, _lib.ie_profile(ctx.handle, int(bool(enable))), "ie_profile")


def ie_profile_read(ctx):
    """Returns {kernel name: (total ms, launches)} for the operator kernels since ie_profile(ctx, True)."""
    ms = np.zeros(len(KERNELS), np.float64)
    cnt = np.zeros(len(KERNELS), np.int32)
    _check(ctx, _lib.ie_profile_read(ctx.handle, _ptr(ms), _ptr(cnt)), "ie_profile_read")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNELS)}


def ie_receiver_fields_table(ctx, e, e0rx, h0):
    """Receiver couplings by reciprocity: e [n_src][3][nz][ny][nx] and e0rx [n_rxdip][3][nz][ny][nx]
    CUDA complex128 tensors; h0 host complex128 [n_src][n_rxdip].  Returns [n_src][n_rxdip]."""
    h0 = np.ascontiguousarray(np.asarray(h0, np.complex128).reshape(ctx.n_src, -1))
    out = np.zeros_like(h0)
    _check(ctx, _lib.ie_receiver_fields_table(ctx.handle, _ptr(e), int(h0.shape[1]), _ptr(e0rx), _ptr(h0), _ptr(out)),
           "ie_receiver_fields_table")
    return out


def ie_get_layer_spectrum(ctx, box=None):
    """Packed layered spectra [(by+1)(bx+1)][3bz][3bz] (layered contexts)."""
    if box is None:
        nx, ny, nz = ctx.grid.nx, ctx.grid.ny, ctx.grid.nz
    else:
        nx, ny, nz = box[1] - box[0], box[3] - box[2], box[5] - box[4]
    out = np.zeros(((ny + 1) * (nx + 1), 3 * nz, 3 * nz), np.complex128)
    _check(ctx, _lib.ie_get_layer_spectrum(ctx.handle, _box(box), _ptr(out)), "ie_get_layer_spectrum")
    return out
