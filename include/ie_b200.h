/*
 * ie_b200.h -- C-ABI of the B200 (sm_100a) integral-equation forward solver with
 * domain-decomposition preconditioning (arXiv 2306.17537).
 *
 * Citations are PAPER.md line numbers ("P:n") with the equation they belong to.
 *
 * The solver computes the total electric field E of the discretised volume IE
 *     (I - G dsigma) E = E0                                   (Eq. 8)
 * on a uniform grid of cells (method of moments), applying G by a 2x zero-padded
 * FFT convolution with the six unique components of the background Green's tensor
 * (Eq. 10), and solves it by restarted GMRES either on the full domain or
 * inside the block Jacobi / block Gauss-Seidel fixed-point iteration of Algorithm 1
 * (Eqs. 19-24), then evaluates receiver magnetic fields (Eq. 4).
 *
 * Conventions shared by every entry point
 *  - Precision: IEEE binary64 / complex128 throughout (interleaved re, im doubles).
 *  - Cells are indexed (i, j, k) along (x, y, z); centroid(i,j,k) = origin + (i dx, j dy, k dz).
 *  - Vector fields (E, E0, operator inputs/outputs) are complex128 arrays
 *        [nrhs][3][nz][ny][nx]   (component-major, x fastest, contiguous),
 *    restricted to the operator's domain (whole grid, or a box; then nx,ny,nz are the
 *    box extents).  Pointers named *_dev are CUDA device pointers, 16-byte aligned.
 *  - Each grid dimension must be a power of two between 1 and 512 (FFT lengths 2..1024);
 *    box extents likewise.  Other sizes return IE_ERR_INVALID_ARGUMENT.
 *  - Ownership: the caller owns every buffer it passes.  The library owns the context
 *    and the persistent per-context data it allocates (Green spectra, dsigma, E0,
 *    twiddle tables); all scratch (FFT intermediates, Krylov bases, DD fields) comes from
 *    the caller-provided workspace (ie_bind_workspace).  The library never frees caller
 *    memory.
 *  - Streams: all device work is enqueued on the stream given to ie_create.
 *    ie_apply_operator is asynchronous; solves and receiver evaluation synchronise the
 *    stream before returning host-visible results.
 *  - Errors: a non-zero ie_status; ie_last_error() returns a message.  No exception or
 *    abort crosses the ABI.  A context is not thread-safe; separate contexts on separate
 *    streams are independent.
 *  - Call order: create -> bind_workspace -> set_contrast -> set_source (or set_incident)
 *    -> apply / solve / receivers.  Violations return IE_ERR_STATE.
 */
#ifndef IE_B200_H
#define IE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ie_ctx ie_ctx; /* opaque; one per (grid, background, frequency) */

typedef enum {
  IE_OK = 0,
  IE_ERR_INVALID_ARGUMENT = 1, /* bad size, pointer, layout, non-symmetric sigma, ... */
  IE_ERR_OUT_OF_MEMORY = 2,    /* device allocation failed, or workspace too small (message has bytes) */
  IE_ERR_CUDA = 3,             /* a CUDA runtime call failed (message has the CUDA error string) */
  IE_ERR_NOT_CONVERGED = 4,    /* solver hit its caps; outputs hold the best iterate, stats valid */
  IE_ERR_BREAKDOWN = 5,        /* non-finite values in a Krylov recurrence */
  IE_ERR_STATE = 6,            /* call-order violation (e.g. no contrast set yet) */
  IE_ERR_PLACEMENT = 7,        /* a source within 1e-6*h of a cell centroid (E0 singular there) */
  IE_ERR_UNSUPPORTED = 8       /* the call does not apply to this context (e.g. set_source on a layered one) */
} ie_status;

/* Uniform grid.  origin = centroid of cell (0,0,0), metres; dx,dy,dz > 0 in metres. */
typedef struct {
  int32_t nx, ny, nz;
  double dx, dy, dz;
  double origin[3];
} ie_grid;

/* Background medium.  The paper uses a homogeneous isotropic background sigma0:
 * n_layers = 1, sigma[0] = sigma0 > 0 (S/m), z_iface = NULL, table = NULL, table_format 0.
 *
 * Layered backgrounds (beyond the paper; DESIGN.md readings
 * R17-R19): the kernel is translation invariant in x and y only,
 *     (G J)_p(i,j,k) = sum_{q,i',j',k'} T_pq(i-i', j-j'; k, k') J_q(i',j',k'),
 * and dsigma = sigma - sigma_b(z_k) I with sigma_b(z) the conductivity of the layer that holds
 * the cell centroid (layer l: z_iface[l-1] <= z < z_iface[l], layers bottom to top).
 *  - table_format 1 (IE_TABLE_QUADRANT): table = HOST complex128 [9][nz][nz][ny][nx],
 *    T[p*3+q][k][k'][dj][di] for offsets di, dj >= 0 (kernel samples including dv and the
 *    self term, like K(d) of the homogeneous kernel); negative offsets follow the mirror
 *    rules T_pq(-di,dj) = sx_p sx_q T_pq(di,dj), sx = (-1,1,1), and T_pq(di,-dj) =
 *    sy_p sy_q T_pq(di,dj), sy = (1,-1,1) (so the stored xy, xz entries at di = 0 and xy, yz
 *    entries at dj = 0 are taken as 0).  Read (copied to the device) inside ie_create.
 *    n_layers > 1 requires this format; then E0 is caller-supplied (ie_set_incident) and
 *    receivers use ie_receiver_fields_table (ie_set_source / ie_receiver_fields return
 *    UNSUPPORTED).
 *  - table_format 2 (IE_TABLE_HOMOGENEOUS): n_layers = 1, table = NULL: the library builds the
 *    degenerate equal-layer table T = K(di, dj, k - k') of sigma[0] itself and runs the
 *    layered operator path on it (same operator as format 0 up to rounding). */
typedef enum { IE_TABLE_NONE = 0, IE_TABLE_QUADRANT = 1, IE_TABLE_HOMOGENEOUS = 2 } ie_table_format;
typedef struct {
  int32_t n_layers;
  const double* sigma;   /* [n_layers], bottom to top, S/m, > 0 */
  const double* z_iface; /* [n_layers-1] ascending, m (NULL when n_layers = 1) */
  const void* table;     /* host table (format 1) or NULL */
  int32_t table_format;  /* ie_table_format */
} ie_background;

/* Rectangular sub-domain Omega_j (Eq. 11): half-open cell ranges. */
typedef struct {
  int32_t i0, i1, j0, j1, k0, k1;
} ie_box;

/* Create a context: validates the grid, computes k0 = sqrt(i omega mu0 sigma0) (Eq. 7),
 * samples the discrete kernel K(d) = G^E(d h) dv (Eq. 5 at centroid offsets, midpoint rule)
 * with the equivolume-sphere self term K(0) = (1/sigma0)[(2/3)(1 - i k0 a) e^{i k0 a} - 1] I,
 * a = (3 dv / 4 pi)^{1/3} (reading R3), and precomputes its 2x-padded FFT
 * (Eq. 10, "pre-calculated before calling the iterative solvers") on the device.
 * cuda_stream: a cudaStream_t (NULL = legacy default stream).  freq_hz > 0.
 * Layered backgrounds (table_format != 0): the table is copied to the device and its
 * 2x-padded x-y spectra are packed per horizontal wavenumber (see ie_get_layer_spectrum).
 * Errors: INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA. */
ie_status ie_create(const ie_grid* grid, const ie_background* bg, double freq_hz, void* cuda_stream,
                    ie_ctx** out);
ie_status ie_destroy(ie_ctx* ctx); /* frees library-owned memory; NULL is a no-op */
const char* ie_last_error(const ie_ctx* ctx); /* never NULL; "" if no error; ctx may be NULL */

/* Scratch bytes needed for the largest call planned: full-domain operations on nrhs right-hand
 * sides with GMRES(restart), and DD over the given boxes (n_boxes may be 0).  The returned
 * size serves every entry point for nrhs <= the given value. */
ie_status ie_workspace_query(ie_ctx* ctx, const ie_box* boxes, int32_t n_boxes, int32_t nrhs, int32_t restart,
                             size_t* bytes);
/* Bind caller-owned device scratch (e.g. torch.empty(bytes, dtype=uint8, device="cuda")).
 * dptr must be 256-byte aligned and stay valid until rebound or ie_destroy. */
ie_status ie_bind_workspace(ie_ctx* ctx, void* dptr, size_t bytes);

/* Conductivity per cell (total sigma, S/m); the library forms dsigma = sigma - sigma0 I
 * on the device.  layout 0 = FULL9: float64 [nz][ny][nx][3][3] row-major, symmetry
 * sigma_pq = sigma_qp checked to 1e-12 relative (else INVALID_ARGUMENT);
 * layout 1 = SYM6: float64 [6][nz][ny][nx], components (xx, yy, zz, xy, xz, yz).
 * sigma_dev is a device pointer; it is read before the call returns. */
ie_status ie_set_contrast(ie_ctx* ctx, const void* sigma_dev, int32_t layout);

/* Magnetic-dipole sources (the tool transmitters).  pos, moment: host arrays
 * [n_src][3] in m and A m^2.  Computes on the device the background field of each source at
 * every centroid, E0 = i omega mu0 g(R)(i k0 - 1/R)(Rhat x m), R = r - r_s (reading R4),
 * kept in library memory as the right-hand sides [n_src][3][nz][ny][nx].
 * Errors: PLACEMENT if a source is within 1e-6*min(dx,dy,dz) of a centroid. */
ie_status ie_set_source(ie_ctx* ctx, int32_t n_src, const double* pos, const double* moment);
/* Copy E0 [n_src][3][nz][ny][nx] into e0_dev (asynchronous). */
ie_status ie_get_incident(ie_ctx* ctx, void* e0_dev);
/* Use a caller-supplied E0 (device, [n_src][3][nz][ny][nx]) instead of set_source; copied. */
ie_status ie_set_incident(ie_ctx* ctx, int32_t n_src, const void* e0_dev);

/* y = (I - G^(box) dsigma^(box)) x  (Eq. 8; for a box, the diagonal block of Eq. 15).
 * box = NULL means the whole grid.  x_dev, y_dev: [nrhs][3][bz][by][bx] (box extents), must
 * not alias.  Asynchronous on the context stream.  Uses workspace. */
ie_status ie_apply_operator(ie_ctx* ctx, const ie_box* box, int32_t nrhs, const void* x_dev, void* y_dev);

/* Restarted GMRES (Saad 1986).  Stops when the estimated ||b - A x|| / ||b|| <= tol
 * (relative to ||b||, as Eq. 9 is relative to ||E0||); the true residual is recomputed at
 * every restart and at exit.  min_iters >= 1 forces at least that many Arnoldi steps
 * (the DD stall guard, reading R10).  Orthogonalisation: classical Gram-Schmidt with
 * DGKS re-orthogonalisation, fused device reductions. */
typedef struct {
  int32_t restart;   /* Krylov dimension m before restart, 1..128 */
  int32_t max_iters; /* cap on A v products */
  int32_t min_iters; /* >= 0 */
  double tol;        /* relative residual target, > 0 */
} ie_gmres_opts;

/* Right preconditioner of every subsequent GMRES on this context (ie_solve_subdomain, the
 * sub-domain and full-domain solves of ie_solve_dd): kind 0 = none, the paper's conventional IE
 * (the default); kind 1 = the contraction-IE right preconditioner P = 2 sigma_b (sigma +
 * sigma_b I)^-1 per cell (Hursan & Zhdanov; the paper's remedy for high contrast):
 * GMRES on (I - G dsigma) P chi = E0, E = P chi -- same solution, same Eq. 9 residual (SURVEY
 * 8(f)-2), built lazily from the contrast.  INVALID_ARGUMENT for other kinds. */
ie_status ie_set_preconditioner(ie_ctx* ctx, int32_t kind);
typedef struct {
  int32_t iters, restarts, converged;
  double relres_est, relres_true;
} ie_solve_stats;

/* Solve (I - G^(box) dsigma^(box)) x = b for each of nrhs right-hand sides (batched on the
 * device).  b_dev, x_dev: [nrhs][3][bz][by][bx]; x_dev holds the initial guess on entry and
 * the solution on exit.  stats: host array [nrhs].  Synchronous.
 * Returns NOT_CONVERGED (x = best iterate) if any system hit max_iters. */
ie_status ie_solve_subdomain(ie_ctx* ctx, const ie_box* box, int32_t nrhs, const void* b_dev, void* x_dev,
                             const ie_gmres_opts* opts, ie_solve_stats* stats);

/* IE_DD_FGMRES_*: Krylov-accelerated DD (the paper's future work):
 * flexible GMRES(10) on the full system, right-preconditioned by one block-Jacobi or block
 * Gauss-Seidel sweep from zero with inner GMRES to inner_tol_fixed; max_sweeps caps the outer
 * (preconditioned) iterations, adaptive / inner_tol_factor are unused. */
typedef enum {
  IE_DD_FULL = 0,
  IE_DD_JACOBI = 1,
  IE_DD_GAUSS_SEIDEL = 2,
  IE_DD_FGMRES_JACOBI = 3,
  IE_DD_FGMRES_GAUSS_SEIDEL = 4
} ie_dd_scheme;

/* Algorithm 1 options.  boxes: a non-overlapping partition of the grid (Eq. 11), host
 * array; Gauss-Seidel visits them in the given order (reading R12).  The inner GMRES
 * threshold is e * inner_tol_factor (adaptive, "threshold = e/10") or
 * inner_tol_fixed; warm start x0 = E^(i),k.  Iteration stops when the full-domain
 * relative residual e (Eq. 9, recomputed after every sweep, reading R9) <= outer_tol, after
 * max_sweeps, or when e grows for 3 consecutive sweeps (NOT_CONVERGED).
 * scheme = IE_DD_FULL ignores the boxes and runs full-domain GMRES with tol = outer_tol. */
typedef struct {
  ie_dd_scheme scheme;
  const ie_box* boxes;
  int32_t n_boxes;
  double outer_tol;
  int32_t adaptive;        /* 1: threshold = e * inner_tol_factor; 0: inner_tol_fixed */
  double inner_tol_fixed;
  double inner_tol_factor; /* 0.1 in the paper */
  int32_t max_sweeps;
  ie_gmres_opts inner;     /* restart, max_iters per sub-domain solve, min_iters (>= 1) */
} ie_dd_opts;

/* Caller-provided stats.  e_hist: host [max_sweeps+1][n_src] (may be NULL);
 * iters: host [max_sweeps][n_boxes][n_src] inner GMRES iterations (may be NULL). */
typedef struct {
  int32_t sweeps, total_inner_iters, full_applies, sub_applies;
  double e_final; /* max over sources of the final Eq. 9 residual */
  double* e_hist;
  int32_t* iters;
} ie_dd_stats;

/* Solve for all n_src sources set by ie_set_source / ie_set_incident, starting from E0
 * (Algorithm 1 "initialize E^0 := E^(0)").  e_dev: [n_src][3][nz][ny][nx], the total
 * field on exit.  Synchronous. */
ie_status ie_solve_dd(ie_ctx* ctx, const ie_dd_opts* opts, void* e_dev, ie_dd_stats* stats);
/* The same with a caller-supplied initial iterate: e_dev holds it on entry (warm start, e.g. the
 * previous tool position), the total field on exit. */
ie_status ie_solve_dd_warm(ie_ctx* ctx, const ie_dd_opts* opts, void* e_dev, ie_dd_stats* stats);

/* Magnetic field at receiver points for every source (Eq. 4):
 * H(r) = H0(r) + sum_c grad g(r - r_c) x (dsigma_c E_c) dv   (G^H of Eq. 6 applied to J),
 * H0 = (k0^2 + grad grad) g m; a cell whose centroid coincides with r contributes 0.
 * e_dev: [n_src][3][nz][ny][nx]; rx_pos: host [n_rx][3]; h_host: host complex128
 * [n_src][n_rx][3].  v_host (optional, may be NULL): i omega mu0 H, i.e. the EMF of unit
 * receiver coils along x, y, z (reading R14).  Synchronous. */
ie_status ie_receiver_fields(ie_ctx* ctx, const void* e_dev, int32_t n_rx, const double* rx_pos, void* h_host,
                             void* v_host);

/* Layered backgrounds: receiver couplings by reciprocity (Eq. 4 with the reciprocity of the
 * discrete system; R17):
 *   h[s][r] = h0[s][r] + (i omega mu0)^-1 sum_c E0rx_r(r_c) . (dsigma_c E_s(r_c)) dv
 * e_dev: [n_src][3][nz][ny][nx] total fields; e0rx_dev: device [n_rxdip][3][nz][ny][nx],
 * background E of the unit receiver dipoles (caller-supplied, like the layered E0);
 * h0_host: host complex128 [n_src][n_rxdip] primary couplings m_r . H0(r_r; source s);
 * h_host: host complex128 [n_src][n_rxdip] out (m_r . H).  Works on every context.
 * Synchronous. */
ie_status ie_receiver_fields_table(ie_ctx* ctx, const void* e_dev, int32_t n_rxdip, const void* e0rx_dev,
                                   const void* h0_host, void* h_host);

/* Introspection for tests / benchmarks. */
typedef struct {
  double k0_re, k0_im;     /* background wavenumber */
  double self_re, self_im; /* K(0) diagonal entry (reading R3) */
  int32_t n_src;
  int32_t kernel_launches; /* number of CUDA kernel launches issued by this context so far */
} ie_info;
ie_status ie_get_info(const ie_ctx* ctx, ie_info* info);
/* Per-kernel device timing of the operator (benchmarks).  enable != 0 starts recording CUDA
 * events around each operator pass on the context stream: k = 0 K-A x-forward+contrast,
 * 1 K-B y-forward, 2 K-C z-convolution, 3 K-D y-inverse, 4 K-E x-inverse+update, 5 K-DE (K-D
 * and K-E fused in one persistent launch), 6 K-AB (K-A and K-B fused in one persistent launch);
 * the fused pairs are opt-in (environment IE_FUSED_DE=1 / IE_FUSED_AB=1 when the context is
 * created; measured slower than the separate passes); enable = 0 stops and clears.  ie_profile_read synchronises the
 * stream and returns, for each slot k, the summed device time ms[k] (milliseconds) and the
 * number of operator applications counts[k] that ran that pass (0 for passes replaced by a
 * fused kernel).  Caller-owned host arrays of 7 entries. */
ie_status ie_profile(ie_ctx* ctx, int32_t enable);
ie_status ie_profile_read(ie_ctx* ctx, double* ms /*[7]*/, int32_t* counts /*[7]*/);
/* Copy the packed Green spectrum of the given box shape (box = NULL: the grid) to the host:
 * complex128 [6][bz+1][by+1][bx+1], components (xx, yy, zz, xy, xz, yz), scaled by
 * 1/(8 bx by bz); entry (kx,ky,kz) of the full padded spectrum F[G_pq] (Eq. 10) is
 * s * packed[c][kz'][ky'][kx'] with k' = min(k, 2n - k) and s = -1 per axis where
 * the component is odd and k > n. */
ie_status ie_get_green_octant(ie_ctx* ctx, const ie_box* box, void* host_out);

/* Layered contexts: copy the packed x-y spectra of the domain (box = NULL: the grid; a box
 * uses the table restricted to its offsets and its layer range) to the host: complex128
 * [(by+1)(bx+1)][3bz][3bz], entry [iy (bx+1) + ix][q bz + k'][p bz + k] =
 * F2[T_pq(., .; k0+k, k0+k')](kx = ix, ky = iy) / (4 bx by), F2 the 2-D DFT of the table
 * circulant-embedded on (2by, 2bx) with the slot at offset +-n set to 0.  The spectrum at a
 * mirrored wavenumber (2bx - ix or 2by - iy) is D M D with D = diag(sx, sy, 1). */
ie_status ie_get_layer_spectrum(ie_ctx* ctx, const ie_box* box, void* host_out);

#ifdef __cplusplus
}
#endif
#endif /* IE_B200_H */
