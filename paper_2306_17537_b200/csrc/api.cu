// C-ABI entry points (include/ie_b200.h) and the domain-decomposition orchestrator
// (Algorithm 1; Eqs. 19-24).
#include <math.h>

#include <algorithm>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ie_internal.h"

static thread_local std::string g_err;  // errors without a context (ie_create)

namespace ie {

ie_status fail(ie_ctx* c, ie_status s, const std::string& msg) {
  if (c) c->err = msg;
  g_err = msg;
  return s;
}
ie_status cuda_fail(ie_ctx* c, cudaError_t e, const char* where) {
  std::string m = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // clear sticky-free errors
  return fail(c, e == cudaErrorMemoryAllocation ? IE_ERR_OUT_OF_MEMORY : IE_ERR_CUDA, m);
}

static long long ncell(const ie_ctx* c) { return (long long)c->g.nx * c->g.ny * c->g.nz; }
constexpr int kFgmresRestart = 10;  // outer FGMRES restart of the Krylov-accelerated DD

static bool box_ok(const ie_ctx* c, const ie_box& b, std::string* why) {
  if (b.i0 < 0 || b.j0 < 0 || b.k0 < 0 || b.i1 > c->g.nx || b.j1 > c->g.ny || b.k1 > c->g.nz || b.i1 <= b.i0 ||
      b.j1 <= b.j0 || b.k1 <= b.k0) {
    *why = "box outside the grid or empty";
    return false;
  }
  if (!is_pow2(b.i1 - b.i0) || !is_pow2(b.j1 - b.j0) || !is_pow2(b.k1 - b.k0)) {
    *why = "box extents must be powers of two";
    return false;
  }
  return true;
}

static ie_box full_box(const ie_ctx* c) { return ie_box{0, c->g.nx, 0, c->g.ny, 0, c->g.nz}; }

static const double* dsig_at(const ie_ctx* c, const ie_box& b) {
  return c->dsig + ((long long)b.k0 * c->g.ny + b.j0) * c->g.nx + b.i0;
}
static const double* at_box(const ie_ctx* c, const double* grid6, const ie_box& b) {
  return grid6 + ((long long)b.k0 * c->g.ny + b.j0) * c->g.nx + b.i0;
}

// a GMRES system on box b; with the contraction-IE right preconditioner (ie_set_preconditioner 1)
// the operator is (I - G dsigma) P, P = 2 sigma_b (sigma + sigma_b I)^-1
static GmresSystem make_sys(const ie_ctx* c, const double2* b_, double2* x_, const ie_box& b, double tol,
                            int min_iters, int precond) {
  GmresSystem s{b_, x_, dsig_at(c, b), tol, min_iters};
  if (precond) {
    s.dsig = at_box(c, c->pre_dp, b);
    s.pm = at_box(c, c->pre_p, b);
    s.pa = at_box(c, c->pre_a, b);
  }
  return s;
}

// Apply on a box-shaped domain for nitems inputs (x[i] compact over the source sub-box src,
// which is relative to the domain box).  y = alpha x + beta G dsigma x (+ y).
static ie_status apply_many(ie_ctx* c, Arena& ar, const ie_box& dom, const ie_box& src,
                            const std::vector<const double2*>& x, const std::vector<double2*>& y, double alpha,
                            double beta, int acc) {
  const int bx = dom.i1 - dom.i0, by = dom.j1 - dom.j0, bz = dom.k1 - dom.k0;
  ie_status st;
  const GreenSpec* gs = green_for(c, bx, by, bz, dom.k0, &st);
  if (!gs) return st;
  const int n = (int)x.size();
  const int items = std::min(n, kMaxItems);
  const size_t mark = ar.used;
  double2* scratch = (double2*)ar.take(apply_scratch_bytes(bx, by, bz, items));
  if (!scratch) {
    ar.used = mark;
    return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for the operator (need " + std::to_string(ar.peak) +
                                             " bytes; see ie_workspace_query)");
  }
  ApplyParams p{};
  p.nx = bx;
  p.ny = by;
  p.nz = bz;
  p.ds_cs = ncell(c);
  p.ds_zs = (long long)c->g.nx * c->g.ny;
  p.ds_ys = c->g.nx;
  p.ghat = gs->oct;
  p.mhat = gs->mhat;
  p.X1 = scratch;
  p.X2 = scratch + (size_t)items * 3 * 2 * bx * by * bz;
  p.alpha = alpha;
  p.beta = beta;
  p.accumulate = acc;
  for (int b0 = 0; b0 < n; b0 += kMaxItems) {
    const int nb = std::min(kMaxItems, n - b0);
    p.n_items = nb;
    for (int i = 0; i < nb; ++i) {
      ApplyItem& it = p.items[i];
      it.x = x[b0 + i];
      it.y = y[b0 + i];
      it.dsig = dsig_at(c, dom);
      it.pm = nullptr;
      it.xscale = 1.0;
      it.xscale_dev = nullptr;
      it.sx0 = src.i0;
      it.sx1 = src.i1;
      it.sy0 = src.j0;
      it.sy1 = src.j1;
      it.sz0 = src.k0;
      it.sz1 = src.k1;
    }
    st = launch_apply(c, p);
    if (st) break;
  }
  ar.used = mark;
  return st;
}

static Arena arena_of(ie_ctx* c) {
  Arena a;
  a.base = c->ws;
  a.cap = c->ws_bytes;
  return a;
}

static size_t dd_bytes(int nx, int ny, int nz, const ie_box* boxes, int n_boxes, int ns, int m) {
  const size_t len = 3ull * nx * ny * nz;
  size_t fixed = 2 * (size_t)ns * len * sizeof(double2) + 3 * (size_t)ns * len * sizeof(double2) + 8192;
  fixed += (2 * kFgmresRestart + 1) * len * sizeof(double2) + 65536;  // Krylov-accelerated DD basis
  // largest same-shape group (Jacobi batch) and any single box (GS)
  std::map<std::vector<int>, int> groups;
  for (int i = 0; i < n_boxes; ++i)
    groups[{boxes[i].i1 - boxes[i].i0, boxes[i].j1 - boxes[i].j0, boxes[i].k1 - boxes[i].k0}]++;
  size_t var = apply_scratch_bytes(nx, ny, nz, std::min(ns, kMaxItems));
  for (auto& g : groups) {
    const int bx = g.first[0], by = g.first[1], bz = g.first[2];
    var = std::max(var, gmres_scratch_bytes(bx, by, bz, g.second * ns, m));
    var = std::max(var, apply_scratch_bytes(bx, by, bz, std::min(g.second * ns, kMaxItems)));
  }
  return fixed + var + 4096;
}

}  // namespace ie

using namespace ie;

extern "C" {

const char* ie_last_error(const ie_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

ie_status ie_create(const ie_grid* g, const ie_background* bg, double freq_hz, void* stream, ie_ctx** out) {
  if (!out) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!g || !bg) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "grid or background is NULL");
  const int n[3] = {g->nx, g->ny, g->nz};
  for (int a = 0; a < 3; ++a)
    if (!is_pow2(n[a]) || n[a] > 512)
      return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "grid dimensions must be powers of two in [1, 512]");
  if (!(g->dx > 0) || !(g->dy > 0) || !(g->dz > 0)) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "cell sizes must be > 0");
  if (!(freq_hz > 0) || !std::isfinite(freq_hz)) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "frequency must be > 0");
  if (bg->n_layers < 1 || !bg->sigma) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "background: n_layers >= 1 and sigma");
  for (int l = 0; l < bg->n_layers; ++l)
    if (!(bg->sigma[l] > 0) || !std::isfinite(bg->sigma[l]))
      return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "background conductivity must be > 0");
  if (bg->n_layers > 1) {
    if (!bg->z_iface) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "layered background needs z_iface");
    for (int l = 1; l < bg->n_layers - 1; ++l)
      if (!(bg->z_iface[l] > bg->z_iface[l - 1])) return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "z_iface must ascend");
    if (bg->table_format != IE_TABLE_QUADRANT || !bg->table)
      return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "a layered background needs a table (table_format 1)");
  }
  if (bg->table_format != IE_TABLE_NONE && bg->table_format != IE_TABLE_QUADRANT &&
      bg->table_format != IE_TABLE_HOMOGENEOUS)
    return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "unknown table_format");
  if ((bg->table_format == IE_TABLE_QUADRANT) != (bg->table != nullptr))
    return fail(nullptr, IE_ERR_INVALID_ARGUMENT, "table pointer and table_format disagree");
  ie_ctx* c = new ie_ctx();
  c->g = *g;
  c->sigma_b = bg->sigma[0];
  c->layered = bg->table_format != IE_TABLE_NONE;
  c->table_format = bg->table_format;
  c->lay_sigma.assign(bg->sigma, bg->sigma + bg->n_layers);
  if (bg->n_layers > 1) c->lay_z.assign(bg->z_iface, bg->z_iface + bg->n_layers - 1);
  c->freq = freq_hz;
  c->omega = 2 * kPi * freq_hz;
  c->stream = (cudaStream_t)stream;
  if (const char* sl = getenv("IE_SLABS")) c->slabs = sl[0] == '1';  // opt-in slab pipeline
  if (const char* fd = getenv("IE_FUSED_DE")) c->fused_de = fd[0] == '1';  // K-DE fused (opt-in)
  if (const char* fa = getenv("IE_FUSED_AB")) c->fused_ab = fa[0] == '1';  // K-AB fused (opt-in)
  if (const char* gd = getenv("IE_GMRES_DEVICE")) c->gmres_device = gd[0] == '1';  // device Arnoldi (opt-in)
  // k0 = sqrt(i omega mu0 sigma0), Re, Im > 0 (Eq. 7)
  c->k0 = std::sqrt(cplx(0.0, c->omega * kMu0 * c->sigma_b));
  // self term K(0) = (1/sigma0)[(2/3)(1 - i k0 a) e^{i k0 a} - 1]  (reading R3)
  const double dv = g->dx * g->dy * g->dz;
  const double a = cbrt(3.0 * dv / (4.0 * kPi));
  const cplx ika = cplx(0.0, 1.0) * c->k0 * a;
  c->self = ((2.0 / 3.0) * (1.0 - ika) * std::exp(ika) - 1.0) / c->sigma_b;
  int dev_count = 0;
  cudaError_t e = cudaGetDeviceCount(&dev_count);
  if (e != cudaSuccess || dev_count == 0) {
    delete c;
    return fail(nullptr, IE_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  ie_status st = build_twiddles(c);
  if (!st && c->layered) st = build_layer_table(c, bg->table);
  if (!st) {
    GreenSpec gs;
    st = c->layered ? build_layer_spec(c, g->nx, g->ny, g->nz, 0, &gs) : build_green(c, g->nx, g->ny, g->nz, &gs);
    if (!st) c->greens.push_back(gs);
  }
  if (st) {
    g_err = c->err;
    ie_destroy(c);
    return st;
  }
  *out = c;
  return IE_OK;
}

ie_status ie_destroy(ie_ctx* c) {
  if (!c) return IE_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  for (auto& g : c->greens) {
    cudaFree(g.oct);
    cudaFree(g.mhat);
  }
  cudaFree(c->tab);
  cudaFree(c->dsig);
  cudaFree(c->pre_p);
  cudaFree(c->e0);
  cudaFree(c->tw.dev);
  cudaFree(c->d_red);
  cudaFree(c->fused_cnt);
  if (c->h_red) cudaFreeHost(c->h_red);
  if (c->h_arnflag) cudaFreeHost(c->h_arnflag);
  for (auto ev : c->ev_arn) cudaEventDestroy(ev);
  for (auto ev : c->ev_pool) cudaEventDestroy(ev);
  if (c->aux_ready) {
    for (auto st : c->aux) cudaStreamDestroy(st);
    for (auto ev : c->aux_ev)
      if (ev) cudaEventDestroy(ev);
  }
  delete c;
  return IE_OK;
}

ie_status ie_workspace_query(ie_ctx* c, const ie_box* boxes, int32_t n_boxes, int32_t nrhs, int32_t restart,
                             size_t* bytes) {
  if (!c || !bytes || nrhs < 1 || restart < 1 || restart > 128 || n_boxes < 0 || (n_boxes > 0 && !boxes))
    return fail(c, IE_ERR_INVALID_ARGUMENT, "workspace_query: bad arguments");
  const int nx = c->g.nx, ny = c->g.ny, nz = c->g.nz;
  size_t b = apply_scratch_bytes(nx, ny, nz, std::min(nrhs, kMaxItems));
  b = std::max(b, gmres_scratch_bytes(nx, ny, nz, nrhs, restart));
  if (n_boxes > 0) b = std::max(b, dd_bytes(nx, ny, nz, boxes, n_boxes, nrhs, restart));
  b = std::max(b, (size_t)(296 + 64 * nrhs) * 3 * sizeof(double2));
  *bytes = b + 65536;
  return IE_OK;
}

ie_status ie_bind_workspace(ie_ctx* c, void* dptr, size_t bytes) {
  if (!c || (!dptr && bytes)) return fail(c, IE_ERR_INVALID_ARGUMENT, "bind_workspace: bad arguments");
  if (((uintptr_t)dptr) & 255) return fail(c, IE_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  c->ws = (char*)dptr;
  c->ws_bytes = bytes;
  return IE_OK;
}

ie_status ie_set_contrast(ie_ctx* c, const void* sigma_dev, int32_t layout) {
  if (!c || !sigma_dev || (layout != 0 && layout != 1))
    return fail(c, IE_ERR_INVALID_ARGUMENT, "set_contrast: bad arguments (layout 0 = FULL9, 1 = SYM6)");
  return pack_contrast(c, sigma_dev, layout);
}

ie_status ie_set_source(ie_ctx* c, int32_t n_src, const double* pos, const double* moment) {
  if (!c || n_src < 1 || !pos || !moment) return fail(c, IE_ERR_INVALID_ARGUMENT, "set_source: bad arguments");
  if (c->lay_sigma.size() > 1)
    return fail(c, IE_ERR_UNSUPPORTED, "set_source: the layered E0 is caller-supplied (ie_set_incident)");
  const long long N = ncell(c);
  if (c->e0 && c->n_src != n_src) {
    cudaFree(c->e0);
    c->e0 = nullptr;
  }
  if (!c->e0) IE_CUDA(c, cudaMalloc(&c->e0, (size_t)n_src * 3 * N * sizeof(double2)));
  c->n_src = n_src;
  ie_status st = compute_incident(c, n_src, pos, moment, c->e0);
  if (st) {
    c->n_src = 0;
    return st;
  }
  // remember sources for H0 at the receivers
  c->err.clear();
  c->src_pos.assign(pos, pos + 3 * n_src);
  c->src_mom.assign(moment, moment + 3 * n_src);
  return IE_OK;
}

ie_status ie_get_incident(ie_ctx* c, void* e0_dev) {
  if (!c || !e0_dev) return fail(c, IE_ERR_INVALID_ARGUMENT, "get_incident: bad arguments");
  if (!c->e0 || c->n_src == 0) return fail(c, IE_ERR_STATE, "no sources set");
  IE_CUDA(c, cudaMemcpyAsync(e0_dev, c->e0, (size_t)c->n_src * 3 * ncell(c) * sizeof(double2),
                             cudaMemcpyDeviceToDevice, c->stream));
  return IE_OK;
}

ie_status ie_set_incident(ie_ctx* c, int32_t n_src, const void* e0_dev) {
  if (!c || n_src < 1 || !e0_dev) return fail(c, IE_ERR_INVALID_ARGUMENT, "set_incident: bad arguments");
  const long long N = ncell(c);
  if (c->e0 && c->n_src != n_src) {
    cudaFree(c->e0);
    c->e0 = nullptr;
  }
  if (!c->e0) IE_CUDA(c, cudaMalloc(&c->e0, (size_t)n_src * 3 * N * sizeof(double2)));
  IE_CUDA(c, cudaMemcpyAsync(c->e0, e0_dev, (size_t)n_src * 3 * N * sizeof(double2), cudaMemcpyDeviceToDevice,
                             c->stream));
  c->n_src = n_src;
  c->src_pos.clear();
  c->src_mom.clear();
  return IE_OK;
}

ie_status ie_apply_operator(ie_ctx* c, const ie_box* box, int32_t nrhs, const void* x_dev, void* y_dev) {
  if (!c || nrhs < 1 || !x_dev || !y_dev || x_dev == y_dev)
    return fail(c, IE_ERR_INVALID_ARGUMENT, "apply_operator: bad arguments");
  if (!c->contrast_set) return fail(c, IE_ERR_STATE, "apply_operator before set_contrast");
  const ie_box b = box ? *box : full_box(c);
  std::string why;
  if (!box_ok(c, b, &why)) return fail(c, IE_ERR_INVALID_ARGUMENT, why);
  const long long nb = 3LL * (b.i1 - b.i0) * (b.j1 - b.j0) * (b.k1 - b.k0);
  std::vector<const double2*> x;
  std::vector<double2*> y;
  for (int r = 0; r < nrhs; ++r) {
    x.push_back((const double2*)x_dev + r * nb);
    y.push_back((double2*)y_dev + r * nb);
  }
  Arena ar = arena_of(c);
  const ie_box src{0, b.i1 - b.i0, 0, b.j1 - b.j0, 0, b.k1 - b.k0};
  return apply_many(c, ar, b, src, x, y, 1.0, -1.0, 0);
}

ie_status ie_solve_subdomain(ie_ctx* c, const ie_box* box, int32_t nrhs, const void* b_dev, void* x_dev,
                             const ie_gmres_opts* o, ie_solve_stats* stats) {
  if (!c || nrhs < 1 || !b_dev || !x_dev || !o || !stats || o->restart < 1 || o->restart > 128 || !(o->tol > 0))
    return fail(c, IE_ERR_INVALID_ARGUMENT, "solve_subdomain: bad arguments");
  if (!c->contrast_set) return fail(c, IE_ERR_STATE, "solve before set_contrast");
  if (c->precond_kind) {
    ie_status sp = ensure_precond(c);
    if (sp) return sp;
  }
  const ie_box b = box ? *box : full_box(c);
  std::string why;
  if (!box_ok(c, b, &why)) return fail(c, IE_ERR_INVALID_ARGUMENT, why);
  const int bx = b.i1 - b.i0, by = b.j1 - b.j0, bz = b.k1 - b.k0;
  const long long nb = 3LL * bx * by * bz;
  std::vector<GmresSystem> sys;
  for (int r = 0; r < nrhs; ++r)
    sys.push_back(make_sys(c, (const double2*)b_dev + r * nb, (double2*)x_dev + r * nb, b, o->tol, o->min_iters,
                           c->precond_kind));
  Arena ar = arena_of(c);
  std::vector<GmresResult> res;
  ie_status st = gmres_batched(c, ar, bx, by, bz, b.k0, (long long)c->g.nx * c->g.ny, c->g.nx, sys, o->restart,
                               o->max_iters, res, nullptr);
  if (st) return st;
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  bool allc = true, brk = false;
  for (int r = 0; r < nrhs; ++r) {
    stats[r].iters = res[r].iters;
    stats[r].restarts = res[r].restarts;
    stats[r].converged = res[r].converged;
    stats[r].relres_est = res[r].relres_est;
    stats[r].relres_true = res[r].relres_true;
    allc = allc && res[r].converged;
    brk = brk || res[r].breakdown;
  }
  if (brk) return fail(c, IE_ERR_BREAKDOWN, "non-finite values in GMRES");
  if (!allc) return fail(c, IE_ERR_NOT_CONVERGED, "GMRES reached max_iters");
  return IE_OK;
}

// ------------------------------------------------------------------------ Algorithm 1
ie_status ie_set_preconditioner(ie_ctx* c, int32_t kind) {
  if (!c) return fail(c, IE_ERR_INVALID_ARGUMENT, "set_preconditioner: null context");
  if (kind < 0 || kind > 1) return fail(c, IE_ERR_INVALID_ARGUMENT, "set_preconditioner: kind 0 or 1");
  c->precond_kind = kind;
  return IE_OK;
}

static ie_status solve_dd_impl(ie_ctx* c, const ie_dd_opts* o, void* e_dev, int32_t init_from_e, ie_dd_stats* stats);

ie_status ie_solve_dd(ie_ctx* c, const ie_dd_opts* o, void* e_dev, ie_dd_stats* stats) {
  return solve_dd_impl(c, o, e_dev, 0, stats);
}

ie_status ie_solve_dd_warm(ie_ctx* c, const ie_dd_opts* o, void* e_dev, ie_dd_stats* stats) {
  return solve_dd_impl(c, o, e_dev, 1, stats);
}

static ie_status solve_dd_impl(ie_ctx* c, const ie_dd_opts* o, void* e_dev, int32_t init_from_e, ie_dd_stats* stats) {
  if (!c || !o || !e_dev || !stats) return fail(c, IE_ERR_INVALID_ARGUMENT, "solve_dd: bad arguments");
  if (!c->contrast_set || !c->e0 || c->n_src < 1) return fail(c, IE_ERR_STATE, "solve_dd needs contrast and sources");
  if (o->inner.restart < 1 || o->inner.restart > 128 || !(o->outer_tol > 0) || o->max_sweeps < 0)
    return fail(c, IE_ERR_INVALID_ARGUMENT, "solve_dd: bad options");
  if (c->precond_kind) {
    ie_status sp = ensure_precond(c);
    if (sp) return sp;
  }
  const int ns = c->n_src;
  const long long N = ncell(c), len = 3 * N;
  double2* E = (double2*)e_dev;
  const int m = o->inner.restart;
  const ie_box fb = full_box(c);
  stats->sweeps = 0;
  stats->total_inner_iters = 0;
  stats->full_applies = 0;
  stats->sub_applies = 0;
  stats->e_final = 0;
  if (!init_from_e) IE_CUDA(c, cudaMemcpyAsync(E, c->e0, (size_t)ns * len * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  Arena ar = arena_of(c);

  if (o->scheme == IE_DD_FULL) {
    std::vector<GmresSystem> sys;
    for (int r = 0; r < ns; ++r)
      sys.push_back(make_sys(c, c->e0 + r * len, E + r * len, fb, o->outer_tol, o->inner.min_iters, c->precond_kind));
    std::vector<GmresResult> res;
    long long ap = 0;
    ie_status st = gmres_batched(c, ar, c->g.nx, c->g.ny, c->g.nz, 0, (long long)c->g.nx * c->g.ny, c->g.nx, sys, m,
                                 o->inner.max_iters, res, &ap);
    if (st) return st;
    bool allc = true, brk = false;
    for (int r = 0; r < ns; ++r) {
      stats->total_inner_iters += res[r].iters;
      stats->e_final = std::max(stats->e_final, res[r].relres_true);
      if (stats->e_hist) stats->e_hist[r] = res[r].relres_true;
      allc = allc && res[r].converged;
      brk = brk || res[r].breakdown;
    }
    stats->full_applies = (int)ap;
    if (brk) return fail(c, IE_ERR_BREAKDOWN, "non-finite values in GMRES");
    if (!allc) return fail(c, IE_ERR_NOT_CONVERGED, "full-domain GMRES reached max_iters");
    return IE_OK;
  }
  if (o->scheme != IE_DD_JACOBI && o->scheme != IE_DD_GAUSS_SEIDEL && o->scheme != IE_DD_FGMRES_JACOBI &&
      o->scheme != IE_DD_FGMRES_GAUSS_SEIDEL)
    return fail(c, IE_ERR_INVALID_ARGUMENT, "solve_dd: unknown scheme");
  const int M = o->n_boxes;
  if (M < 1 || !o->boxes) return fail(c, IE_ERR_INVALID_ARGUMENT, "solve_dd: no boxes");
  // partition check (Eq. 11): non-overlapping cover of the grid
  {
    std::vector<unsigned char> cover(N, 0);
    for (int i = 0; i < M; ++i) {
      std::string why;
      if (!box_ok(c, o->boxes[i], &why)) return fail(c, IE_ERR_INVALID_ARGUMENT, "box " + std::to_string(i) + ": " + why);
      const ie_box& b = o->boxes[i];
      for (int k = b.k0; k < b.k1; ++k)
        for (int j = b.j0; j < b.j1; ++j)
          for (int x = b.i0; x < b.i1; ++x) cover[((long long)k * c->g.ny + j) * c->g.nx + x]++;
    }
    for (long long i = 0; i < N; ++i)
      if (cover[i] != 1) return fail(c, IE_ERR_INVALID_ARGUMENT, "boxes must partition the grid (Eq. 11)");
  }
  // persistent DD buffers
  double2* S = (double2*)ar.take((size_t)ns * len * sizeof(double2));  // coupling field G dsigma E
  double2* T = (double2*)ar.take((size_t)ns * len * sizeof(double2));  // E0 + S
  double2* Bb = (double2*)ar.take((size_t)ns * len * sizeof(double2)); // per-box rhs   [box][rhs][3Nb]
  double2* Xb = (double2*)ar.take((size_t)ns * len * sizeof(double2)); // per-box x
  double2* Ob = (double2*)ar.take((size_t)ns * len * sizeof(double2)); // per-box old x / delta
  if (!S || !T || !Bb || !Xb || !Ob)
    return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for DD (see ie_workspace_query with the boxes)");
  std::vector<long long> boff(M);  // offset of box i's [rhs][3Nb] block
  {
    long long off = 0;
    for (int i = 0; i < M; ++i) {
      boff[i] = off;
      const ie_box& b = o->boxes[i];
      off += (long long)ns * 3 * (b.i1 - b.i0) * (b.j1 - b.j0) * (b.k1 - b.k0);
    }
  }
  auto nbox = [&](int i) {
    const ie_box& b = o->boxes[i];
    return 3LL * (b.i1 - b.i0) * (b.j1 - b.j0) * (b.k1 - b.k0);
  };
  std::vector<double> e0n(ns), e(ns), eprev(ns);
  std::vector<int> grow(ns, 0);
  std::vector<char> active(ns, 1);
  ie_status st = norms2(c, c->e0, nullptr, ns, len, len, e0n.data());
  if (st) return st;
  for (int r = 0; r < ns; ++r) e0n[r] = sqrt(e0n[r]);

  auto full_G = [&](const std::vector<int>& rr) -> ie_status {  // S_r = G dsigma E_r
    std::vector<const double2*> x;
    std::vector<double2*> y;
    for (int r : rr) {
      x.push_back(E + r * len);
      y.push_back(S + r * len);
    }
    stats->full_applies += (int)rr.size();
    return apply_many(c, ar, fb, fb, x, y, 0.0, 1.0, 0);
  };
  auto residual = [&](const std::vector<int>& rr) -> ie_status {  // T = E0 + S; e = ||T - E|| / ||E0||
    for (int r : rr) {
      launch_axpby(c, T + r * len, 1.0, c->e0 + r * len, 1.0, S + r * len, len);
      double v;
      ie_status s2 = norms2(c, T + r * len, E + r * len, 1, len, 0, &v);
      if (s2) return s2;
      e[r] = e0n[r] > 0 ? sqrt(v) / e0n[r] : 0.0;
    }
    return IE_OK;
  };
  std::vector<int> all;
  for (int r = 0; r < ns; ++r) all.push_back(r);
  st = full_G(all);
  if (st) return st;
  st = residual(all);
  if (st) return st;
  for (int r = 0; r < ns; ++r) {
    if (stats->e_hist) stats->e_hist[r] = e[r];
    active[r] = e[r] > o->outer_tol;
  }
  bool diverged = false, breakdown = false;
  // rhs b_i = T|_i - G_ii dsigma_i E|_i for boxes in `ids` and rhs in `rr`; x0 = E|_i
  auto assemble = [&](const std::vector<int>& ids, const std::vector<int>& rr) -> ie_status {
    for (int i : ids) {
      const ie_box& b = o->boxes[i];
      for (int r : rr) {
        double2* bb = Bb + boff[i] + r * nbox(i);
        double2* xb = Xb + boff[i] + r * nbox(i);
        double2* ob = Ob + boff[i] + r * nbox(i);
        launch_gather(c, T + r * len, bb, b, 1, 0, 0);
        launch_gather(c, E + r * len, ob, b, 1, 0, 0);
        launch_axpby(c, xb, 1.0, ob, 0.0, nullptr, nbox(i));
      }
      std::vector<const double2*> x;
      std::vector<double2*> y;
      for (int r : rr) {
        x.push_back(Ob + boff[i] + r * nbox(i));
        y.push_back(Bb + boff[i] + r * nbox(i));
      }
      const ie_box src{0, b.i1 - b.i0, 0, b.j1 - b.j0, 0, b.k1 - b.k0};
      stats->sub_applies += (int)rr.size();
      ie_status s2 = apply_many(c, ar, b, src, x, y, 0.0, -1.0, 1);
      if (s2) return s2;
    }
    return IE_OK;
  };
  auto solve_boxes = [&](const std::vector<int>& ids, const std::vector<int>& rr, int sweep) -> ie_status {
    // all boxes in ids share one shape
    const ie_box& b0 = o->boxes[ids[0]];
    std::vector<GmresSystem> sys;
    std::vector<std::pair<int, int>> who;
    for (int i : ids)
      for (int r : rr) {
        const double thr = o->adaptive ? e[r] * o->inner_tol_factor : o->inner_tol_fixed;
        sys.push_back(make_sys(c, Bb + boff[i] + r * nbox(i), Xb + boff[i] + r * nbox(i), o->boxes[i], thr,
                               std::max(1, o->inner.min_iters), c->precond_kind));
        who.push_back({i, r});
      }
    std::vector<GmresResult> res;
    const size_t mark = ar.used;
    long long ap = 0;
    ie_status s2 = gmres_batched(c, ar, b0.i1 - b0.i0, b0.j1 - b0.j0, b0.k1 - b0.k0, b0.k0, (long long)c->g.nx * c->g.ny,
                                 c->g.nx, sys, m, o->inner.max_iters, res, &ap);
    ar.used = mark;
    if (s2) return s2;
    stats->sub_applies += (int)ap;
    for (size_t t = 0; t < who.size(); ++t) {
      stats->total_inner_iters += res[t].iters;
      if (res[t].breakdown) breakdown = true;
      if (stats->iters) stats->iters[((size_t)sweep * M + who[t].first) * ns + who[t].second] = res[t].iters;
    }
    return IE_OK;
  };
  // group boxes by shape (Jacobi batches)
  std::map<std::vector<int>, std::vector<int>> groups;
  for (int i = 0; i < M; ++i) {
    const ie_box& b = o->boxes[i];
    groups[{b.i1 - b.i0, b.j1 - b.j0, b.k1 - b.k0, c->layered ? b.k0 : 0}].push_back(i);
  }

  // ------------------------------------------------ Krylov-accelerated DD
  // Flexible GMRES(kFgmresRestart) on the full system (I - G dsigma) E = E0, right-
  // preconditioned by one DD sweep from zero (block Jacobi: z_i = A_ii^-1 v_i, batched;
  // block Gauss-Seidel: z_i = A_ii^-1 (v_i + sum_{j<i} (G dsigma z_j)|_i)) with inner GMRES to the
  // fixed tolerance inner_tol_fixed.  The preconditioner changes between applications, hence
  // FGMRES (Saad 1993): the solution update uses the stored preconditioned vectors Z.
  if (o->scheme == IE_DD_FGMRES_JACOBI || o->scheme == IE_DD_FGMRES_GAUSS_SEIDEL) {
    const bool jac = o->scheme == IE_DD_FGMRES_JACOBI;
    const int mo = kFgmresRestart;
    double2* Vb = (double2*)ar.take((size_t)(mo + 1) * len * sizeof(double2));
    double2* Zb = (double2*)ar.take((size_t)mo * len * sizeof(double2));
    if (!Vb || !Zb) return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for the outer FGMRES basis");
    auto Vj = [&](int j) { return Vb + (long long)j * len; };
    auto Zj = [&](int j) { return Zb + (long long)j * len; };
    const double thr = o->inner_tol_fixed;
    // z = M^-1 v for right-hand side r (box buffers of rhs r)
    auto precond_apply = [&](const double2* v, double2* z, int r) -> ie_status {
      std::vector<int> rr1{r};
      if (jac) {
        for (auto& g : groups) {
          for (int i : g.second) {
            launch_gather(c, v, Bb + boff[i] + r * nbox(i), o->boxes[i], 1, 0, 0);
            launch_axpby(c, Xb + boff[i] + r * nbox(i), 0.0, Bb + boff[i] + r * nbox(i), 0.0, nullptr, nbox(i));
          }
          std::vector<GmresSystem> sys;
          for (int i : g.second)
            sys.push_back(make_sys(c, Bb + boff[i] + r * nbox(i), Xb + boff[i] + r * nbox(i), o->boxes[i], thr,
                                   std::max(1, o->inner.min_iters), c->precond_kind));
          const ie_box& b0 = o->boxes[g.second[0]];
          std::vector<GmresResult> res;
          const size_t mark = ar.used;
          long long ap = 0;
          ie_status s2 = gmres_batched(c, ar, b0.i1 - b0.i0, b0.j1 - b0.j0, b0.k1 - b0.k0, b0.k0,
                                       (long long)c->g.nx * c->g.ny, c->g.nx, sys, m, o->inner.max_iters, res, &ap);
          ar.used = mark;
          if (s2) return s2;
          stats->sub_applies += (int)ap;
          for (auto& q : res) {
            stats->total_inner_iters += q.iters;
            if (q.breakdown) breakdown = true;
          }
        }
        for (int i = 0; i < M; ++i) launch_scatter(c, z, Xb + boff[i] + r * nbox(i), o->boxes[i], 1, 0, 0);
        return IE_OK;
      }
      double2* Sr = S + r * len;
      double2* Tr = T + r * len;
      launch_axpby(c, Sr, 0.0, v, 0.0, nullptr, len);
      launch_axpby(c, z, 0.0, v, 0.0, nullptr, len);
      for (int i = 0; i < M; ++i) {
        launch_axpby(c, Tr, 1.0, v, 1.0, Sr, len);  // v + sum_{j<i} G dsigma z_j
        double2* bb = Bb + boff[i] + r * nbox(i);
        double2* xb = Xb + boff[i] + r * nbox(i);
        launch_gather(c, Tr, bb, o->boxes[i], 1, 0, 0);
        launch_axpby(c, xb, 0.0, bb, 0.0, nullptr, nbox(i));
        std::vector<GmresSystem> sys{make_sys(c, bb, xb, o->boxes[i], thr, std::max(1, o->inner.min_iters),
                                              c->precond_kind)};
        const ie_box& b0 = o->boxes[i];
        std::vector<GmresResult> res;
        const size_t mark = ar.used;
        long long ap = 0;
        ie_status s2 = gmres_batched(c, ar, b0.i1 - b0.i0, b0.j1 - b0.j0, b0.k1 - b0.k0, b0.k0,
                                     (long long)c->g.nx * c->g.ny, c->g.nx, sys, m, o->inner.max_iters, res, &ap);
        ar.used = mark;
        if (s2) return s2;
        stats->sub_applies += (int)ap;
        stats->total_inner_iters += res[0].iters;
        if (res[0].breakdown) breakdown = true;
        launch_scatter(c, z, xb, o->boxes[i], 1, 0, 0);
        if (i + 1 < M) {
          stats->full_applies += 1;
          s2 = apply_many(c, ar, fb, o->boxes[i], {xb}, {Sr}, 0.0, 1.0, 1);
          if (s2) return s2;
        }
      }
      return IE_OK;
    };
    int outer = 0;
    for (int r = 0; r < ns; ++r) {
      if (!active[r]) continue;
      double2* x = E + r * len;
      const double bnorm = e0n[r];
      bool done = false;
      int it = 0;
      while (!done && it < o->max_sweeps) {
        // true residual r0 = E0 - A x into V_0
        launch_axpby(c, Vj(0), 1.0, c->e0 + r * len, 0.0, nullptr, len);
        stats->full_applies += 1;
        st = apply_many(c, ar, fb, fb, {x}, {Vj(0)}, -1.0, 1.0, 1);
        if (st) return st;
        double b2;
        st = norms2(c, Vj(0), nullptr, 1, len, 0, &b2);
        if (st) return st;
        const double beta = sqrt(b2);
        e[r] = bnorm > 0 ? beta / bnorm : 0.0;
        if (!std::isfinite(beta)) {
          breakdown = true;
          break;
        }
        if (e[r] <= o->outer_tol || beta == 0.0) {
          done = true;  // e[r] is the true residual
          break;
        }
        launch_axpby(c, Vj(0), 1.0 / beta, Vj(0), 0.0, nullptr, len);
        std::vector<cplx> H((size_t)(mo + 1) * mo, 0.0), cs(mo), sn(mo), g(mo + 1, 0.0), y;
        g[0] = beta;
        int k = 0;
        for (; k < mo && it < o->max_sweeps; ++k) {
          st = precond_apply(Vj(k), Zj(k), r);
          if (st) return st;
          stats->full_applies += 1;
          st = apply_many(c, ar, fb, fb, {Zj(k)}, {Vj(k + 1)}, 1.0, -1.0, 0);  // w = A z_k
          if (st) return st;
          std::vector<cplx> h(k + 1), h2(k + 1);
          double w2, w2b;
          st = vec_dots(c, ar, Vj(k + 1), Vb, k + 1, len, h.data(), &w2);
          if (st) return st;
          std::vector<cplx> neg(k + 1);
          double hs = 0;
          for (int j = 0; j <= k; ++j) {
            neg[j] = -h[j];
            hs += std::norm(h[j]);
          }
          st = vec_axpy(c, ar, Vj(k + 1), Vj(k + 1), Vb, k + 1, neg.data(), len);
          if (st) return st;
          if (w2 - hs < 0.01 * w2) {  // DGKS re-orthogonalisation (eta = 0.1, as the inner GMRES)
            st = vec_dots(c, ar, Vj(k + 1), Vb, k + 1, len, h2.data(), &w2b);
            if (st) return st;
            for (int j = 0; j <= k; ++j) {
              neg[j] = -h2[j];
              h[j] += h2[j];
            }
            st = vec_axpy(c, ar, Vj(k + 1), Vj(k + 1), Vb, k + 1, neg.data(), len);
            if (st) return st;
          }
          double nw2;
          st = norms2(c, Vj(k + 1), nullptr, 1, len, 0, &nw2);
          if (st) return st;
          const double hk1 = sqrt(nw2);
          cplx* Hk = &H[(size_t)k * (mo + 1)];
          for (int j = 0; j <= k; ++j) Hk[j] = h[j];
          Hk[k + 1] = hk1;
          for (int j = 0; j < k; ++j) {
            const cplx t = cs[j] * Hk[j] + sn[j] * Hk[j + 1];
            Hk[j + 1] = -std::conj(sn[j]) * Hk[j] + std::conj(cs[j]) * Hk[j + 1];
            Hk[j] = t;
          }
          const cplx a = Hk[k], bb = Hk[k + 1];
          const double den = sqrt(std::norm(a) + std::norm(bb));
          cs[k] = den == 0.0 ? cplx(1.0) : std::conj(a / den);
          sn[k] = den == 0.0 ? cplx(0.0) : std::conj(bb / den);
          Hk[k] = cs[k] * a + sn[k] * bb;
          Hk[k + 1] = 0.0;
          g[k + 1] = -std::conj(sn[k]) * g[k];
          g[k] = cs[k] * g[k];
          ++it;
          outer = std::max(outer, it);  // stats->sweeps = the largest per-source count
          const double est = std::abs(g[k + 1]) / bnorm;
          if (stats->e_hist && it <= o->max_sweeps) stats->e_hist[(size_t)it * ns + r] = est;
          if (hk1 > 0) launch_axpby(c, Vj(k + 1), 1.0 / hk1, Vj(k + 1), 0.0, nullptr, len);
          if (est <= o->outer_tol || !(hk1 > 1e-14 * std::abs(Hk[k]))) {
            ++k;
            break;
          }
        }
        // x += Z y, y = H^-1 g (upper triangular)
        y.assign(k, 0.0);
        for (int j = k - 1; j >= 0; --j) {
          cplx t = g[j];
          for (int l = j + 1; l < k; ++l) t -= H[(size_t)l * (mo + 1) + j] * y[l];
          y[j] = t / H[(size_t)j * (mo + 1) + j];
        }
        st = vec_axpy(c, ar, x, x, Zb, k, y.data(), len);
        if (st) return st;
      }
      if (!done) {  // final true residual
        launch_axpby(c, T + r * len, 1.0, c->e0 + r * len, 0.0, nullptr, len);
        stats->full_applies += 1;
        st = apply_many(c, ar, fb, fb, {x}, {T + r * len}, -1.0, 1.0, 1);
        if (st) return st;
        double v2;
        st = norms2(c, T + r * len, nullptr, 1, len, 0, &v2);
        if (st) return st;
        e[r] = bnorm > 0 ? sqrt(v2) / bnorm : 0.0;
      }
    }
    IE_CUDA(c, cudaStreamSynchronize(c->stream));
    stats->sweeps = outer;
    bool allc = true;
    for (int r = 0; r < ns; ++r) {
      stats->e_final = std::max(stats->e_final, e[r]);
      allc = allc && e[r] <= o->outer_tol;
    }
    if (breakdown) return fail(c, IE_ERR_BREAKDOWN, "non-finite values in the Krylov-accelerated DD");
    if (!allc) return fail(c, IE_ERR_NOT_CONVERGED, "Krylov-accelerated DD reached max_sweeps outer iterations");
    return IE_OK;
  }

  int sweep = 0;
  while (sweep < o->max_sweeps) {
    std::vector<int> rr;
    for (int r = 0; r < ns; ++r)
      if (active[r]) rr.push_back(r);
    if (rr.empty()) break;
    if (o->scheme == IE_DD_JACOBI) {
      for (auto& g : groups) {
        st = assemble(g.second, rr);
        if (st) return st;
        st = solve_boxes(g.second, rr, sweep);
        if (st) return st;
      }
      for (int i = 0; i < M; ++i)
        for (int r : rr) launch_scatter(c, E + r * len, Xb + boff[i] + r * nbox(i), o->boxes[i], 1, 0, 0);
      st = full_G(rr);
      if (st) return st;
    } else {  // Gauss-Seidel, boxes in the given order
      for (int i = 0; i < M; ++i) {
        for (int r : rr) launch_axpby(c, T + r * len, 1.0, c->e0 + r * len, 1.0, S + r * len, len);
        st = assemble({i}, rr);
        if (st) return st;
        st = solve_boxes({i}, rr, sweep);
        if (st) return st;
        // delta = x_new - x_old on box i; S += G dsigma (delta restricted to box i)
        std::vector<const double2*> x;
        std::vector<double2*> y;
        for (int r : rr) {
          double2* ob = Ob + boff[i] + r * nbox(i);
          launch_axpby(c, ob, 1.0, Xb + boff[i] + r * nbox(i), -1.0, ob, nbox(i));
          x.push_back(ob);
          y.push_back(S + r * len);
          launch_scatter(c, E + r * len, Xb + boff[i] + r * nbox(i), o->boxes[i], 1, 0, 0);
        }
        stats->full_applies += (int)rr.size();
        st = apply_many(c, ar, fb, o->boxes[i], x, y, 0.0, 1.0, 1);
        if (st) return st;
      }
    }
    ++sweep;
    eprev = e;
    st = residual(rr);
    if (st) return st;
    for (int r : rr) {
      grow[r] = e[r] > eprev[r] ? grow[r] + 1 : 0;
      if (!std::isfinite(e[r])) breakdown = true;
      if (grow[r] >= 3) diverged = true;
      active[r] = e[r] > o->outer_tol && std::isfinite(e[r]);
    }
    if (stats->e_hist)
      for (int r = 0; r < ns; ++r) stats->e_hist[(size_t)sweep * ns + r] = e[r];
    if (diverged || breakdown) break;
  }
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  stats->sweeps = sweep;
  bool allc = true;
  for (int r = 0; r < ns; ++r) {
    stats->e_final = std::max(stats->e_final, e[r]);
    allc = allc && e[r] <= o->outer_tol;
  }
  if (breakdown) return fail(c, IE_ERR_BREAKDOWN, "non-finite values in the DD iteration");
  if (!allc) return fail(c, IE_ERR_NOT_CONVERGED, diverged ? "DD residual grew for 3 sweeps" : "DD reached max_sweeps");
  return IE_OK;
}

ie_status ie_receiver_fields(ie_ctx* c, const void* e_dev, int32_t n_rx, const double* rx_pos, void* h_host,
                             void* v_host) {
  if (!c || !e_dev || n_rx < 1 || !rx_pos || !h_host) return fail(c, IE_ERR_INVALID_ARGUMENT, "receiver_fields: bad arguments");
  if (!c->contrast_set || c->n_src < 1) return fail(c, IE_ERR_STATE, "receiver_fields needs contrast and sources");
  if (c->lay_sigma.size() > 1)
    return fail(c, IE_ERR_UNSUPPORTED, "receiver_fields: layered backgrounds use ie_receiver_fields_table");
  if ((int)c->src_pos.size() != 3 * c->n_src)
    return fail(c, IE_ERR_STATE, "receiver_fields needs dipole sources (ie_set_source) for H0");
  Arena ar = arena_of(c);
  double2* scratch = (double2*)ar.take((size_t)(296 + c->n_src * n_rx) * 3 * sizeof(double2));
  if (!scratch) return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for receivers");
  std::vector<cplx> h((size_t)c->n_src * n_rx * 3);
  ie_status st = receivers(c, (const double2*)e_dev, n_rx, rx_pos, h.data(), c->src_pos.data(), c->src_mom.data(),
                           c->n_src, scratch);
  if (st) return st;
  std::memcpy(h_host, h.data(), h.size() * sizeof(cplx));
  if (v_host) {
    cplx* v = (cplx*)v_host;
    const cplx iwm = cplx(0.0, c->omega * kMu0);
    for (size_t i = 0; i < h.size(); ++i) v[i] = iwm * h[i];
  }
  return IE_OK;
}

ie_status ie_get_info(const ie_ctx* c, ie_info* info) {
  if (!c || !info) return IE_ERR_INVALID_ARGUMENT;
  info->k0_re = c->k0.real();
  info->k0_im = c->k0.imag();
  info->self_re = c->self.real();
  info->self_im = c->self.imag();
  info->n_src = c->n_src;
  info->kernel_launches = (int32_t)std::min<long long>(c->launches, 0x7fffffff);
  return IE_OK;
}

ie_status ie_profile(ie_ctx* c, int32_t enable) {
  if (!c) return IE_ERR_INVALID_ARGUMENT;
  c->profiling = enable != 0;
  c->ev_marks.clear();
  c->ev_used = 0;
  return IE_OK;
}

ie_status ie_profile_read(ie_ctx* c, double* ms, int32_t* counts) {
  if (!c || !ms || !counts) return fail(c, IE_ERR_INVALID_ARGUMENT, "profile_read: bad arguments");
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < kProfSlots; ++k) {
    ms[k] = 0;
    counts[k] = 0;
  }
  // per kernel: summed device time of its passes; counts = number of operator applications
  // (a slab-pipelined application runs a kernel once per slab: those passes add to one count)
  int applies = 0;
  for (auto& mk : c->ev_marks) {
    float t = 0;
    IE_CUDA(c, cudaEventElapsedTime(&t, c->ev_pool[mk.ev0], c->ev_pool[mk.ev1]));
    ms[mk.kernel] += t;
    if (mk.kernel == 0 || mk.kernel == kProfFusedAB) ++applies;  // one front pass per application
  }
  // passes that ran: a fused kernel replaces its parts (those report 0 ms, 0 applications)
  std::vector<int> ran(kProfSlots, 0);
  for (auto& mk : c->ev_marks) ran[mk.kernel] = 1;
  for (int k = 0; k < kProfSlots; ++k) counts[k] = ran[k] ? applies : 0;
  return IE_OK;
}

ie_status ie_get_green_octant(ie_ctx* c, const ie_box* box, void* host_out) {
  if (!c || !host_out) return fail(c, IE_ERR_INVALID_ARGUMENT, "get_green_octant: bad arguments");
  const ie_box b = box ? *box : full_box(c);
  std::string why;
  if (!box_ok(c, b, &why)) return fail(c, IE_ERR_INVALID_ARGUMENT, why);
  ie_status st;
  if (c->layered) return fail(c, IE_ERR_STATE, "get_green_octant: layered context (ie_get_layer_spectrum)");
  const GreenSpec* gs = green_for(c, b.i1 - b.i0, b.j1 - b.j0, b.k1 - b.k0, b.k0, &st);
  if (!gs) return st;
  const size_t n = 6ull * (gs->nx + 1) * (gs->ny + 1) * (gs->nz + 1);
  IE_CUDA(c, cudaMemcpyAsync(host_out, gs->oct, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  return IE_OK;
}

ie_status ie_receiver_fields_table(ie_ctx* c, const void* e_dev, int32_t n_rxdip, const void* e0rx_dev,
                                   const void* h0_host, void* h_host) {
  if (!c || !e_dev || n_rxdip < 1 || !e0rx_dev || !h0_host || !h_host)
    return fail(c, IE_ERR_INVALID_ARGUMENT, "receiver_fields_table: bad arguments");
  if (!c->contrast_set || c->n_src < 1) return fail(c, IE_ERR_STATE, "receiver_fields_table needs contrast and sources");
  Arena ar = arena_of(c);
  const size_t pairs = (size_t)c->n_src * n_rxdip;
  const size_t avail = c->ws_bytes > 4096 ? (c->ws_bytes - 4096) / sizeof(double2) : 0;
  const size_t elems = std::min(pairs * 256, avail);
  double2* scratch = elems >= pairs ? (double2*)ar.take(elems * sizeof(double2)) : nullptr;
  if (!scratch) return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for receivers");
  return receivers_table(c, (const double2*)e_dev, n_rxdip, (const double2*)e0rx_dev, (const cplx*)h0_host,
                         (cplx*)h_host, scratch, elems);
}

ie_status ie_get_layer_spectrum(ie_ctx* c, const ie_box* box, void* host_out) {
  if (!c || !host_out) return fail(c, IE_ERR_INVALID_ARGUMENT, "get_layer_spectrum: bad arguments");
  if (!c->layered) return fail(c, IE_ERR_STATE, "get_layer_spectrum: homogeneous context (ie_get_green_octant)");
  const ie_box b = box ? *box : full_box(c);
  std::string why;
  if (!box_ok(c, b, &why)) return fail(c, IE_ERR_INVALID_ARGUMENT, why);
  ie_status st;
  const GreenSpec* gs = green_for(c, b.i1 - b.i0, b.j1 - b.j0, b.k1 - b.k0, b.k0, &st);
  if (!gs) return st;
  const size_t R = 3ull * gs->nz;
  const size_t n = (size_t)(gs->nx + 1) * (gs->ny + 1) * R * R;
  IE_CUDA(c, cudaMemcpyAsync(host_out, gs->mhat, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  return IE_OK;
}

}  // extern "C"
