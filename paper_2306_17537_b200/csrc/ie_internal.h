// Internal declarations shared by the CUDA translation units of libie_b200.so.
// Not part of the C-ABI (that is include/ie_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <complex>
#include <deque>
#include <string>
#include <vector>

#include "../../include/ie_b200.h"

namespace ie {

using cplx = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double kMu0 = 4e-7 * kPi;  // DESIGN.md reading R1
constexpr int kMaxItems = 48;        // batch items per operator launch (kernel-parameter budget)
constexpr int kMaxLog2 = 10;         // FFT lengths 2 .. 1024
constexpr int kProfSlots = 7;        // ie_profile_read: K-A .. K-E, K-DE (fused), K-AB (fused)
constexpr int kProfFusedDE = 5, kProfFusedAB = 6;

// -------------------------------------------------------------------- operator batch
// One operator application on one right-hand side / sub-domain.  The operator's domain is
// an (nx,ny,nz) box; the source (contrast) region is the sub-box [s?0, s?1) of it and the
// input x is compact over that sub-box.  y = alpha*xs*x + beta*conv + (accumulate ? y : 0),
// conv = G (dsigma * xs * x) on the domain, xs = xscale.
struct ApplyItem {
  const double2* x;    // [3][sz][sy][sx] over the source sub-box
  double2* y;          // [3][nz][ny][nx] over the domain
  const double* dsig;  // sym6 dsigma (or dsigma P) at domain cell (0,0,0); strides in ApplyParams
  const double* pm;    // contraction-IE right preconditioner P (sym6, same strides) or null:
                       // the identity term becomes P x (the operator applied is (I - G dsigma) P)
  double xscale;
  const double* xscale_dev;  // if non-null: the scale is *xscale_dev (device-side GMRES basis scales)
  int sx0, sx1, sy0, sy1, sz0, sz1;
};

#ifdef __CUDACC__
__device__ __forceinline__ double item_xscale(const ApplyItem& it) {
  return it.xscale_dev ? *it.xscale_dev : it.xscale;
}
#endif

struct ApplyParams {
  int nx, ny, nz;
  long long ds_cs, ds_zs, ds_ys;  // dsigma strides (doubles): component, z, y (x stride 1)
  const double2* ghat;            // packed spectrum [6][nz+1][ny+1][nx+1]
  double2* X1;                    // [item][3][nz][ny][2nx]
  double2* X2;                    // [item][3][nz][2ny][x2w]
  int x2w, k0x;                   // X2 row width and first kx it holds: (2nx, 0), or a slab
  double alpha, beta;
  int accumulate;
  const double2* tw_x;   // twiddles, L = 2nx, forward radix order
  const double2* tw_y;   // L = 2ny, forward order
  const double2* tw_z;   // L = 2nz, forward order
  const double2* tw_zr;  // L = 2nz, reversed order
  const double2* pw_z;   // exp(-2 pi i m / 2nz), m < 2nz (radix-16 z-pass)
  const double2* mhat;   // layered background: packed z-z' spectra (layered.cu), else null
  int n_items;
  int rev;  // K-B / K-E: CTAs walk their tiles in reverse launch order (set per launch, operator.cu)
  ApplyItem items[kMaxItems];
};

struct Twiddles {
  double2* dev = nullptr;
  int off[kMaxLog2 + 1][2] = {};  // [log2 L][order]
  int pw[kMaxLog2 + 1] = {};      // [log2 L]: exp(-2 pi i m / L), m = 0 .. L-1
  const double2* get(int L, int rev) const;
  const double2* powers(int L) const;
};

struct GreenSpec {
  int nx, ny, nz;
  int k0 = 0;               // layered: first cell layer of the domain (the spectra depend on it)
  double2* oct = nullptr;   // homogeneous: [6][nz+1][ny+1][nx+1]
  double2* mhat = nullptr;  // layered: [(ny+1)(nx+1)][3nz (q,k')][3nz (p,k)] (layered.cu)
};

// workspace bump allocator (caller-owned memory)
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0, peak = 0;
  bool counting = false;  // size-query mode: no memory, only accounting
  void* take(size_t bytes);
};

}  // namespace ie

struct ie_ctx {
  ie_grid g;
  double sigma_b = 0, freq = 0, omega = 0;
  ie::cplx k0, self;
  cudaStream_t stream = nullptr;
  ie::Twiddles tw;
  std::deque<ie::GreenSpec> greens;  // [0] = whole grid (deque: stable element addresses)
  double* dsig = nullptr;             // sym6 [6][nz][ny][nx]
  // layered background (readings R17-R19): table of kernel samples on the
  // device, quadrant offsets [9][nz][nz][ny][nx]; per-layer conductivities
  bool layered = false;
  int table_format = 0;
  std::vector<double> lay_sigma, lay_z;  // [n_layers], [n_layers-1]
  double2* tab = nullptr;
  double2* e0 = nullptr;
  int n_src = 0;
  std::vector<double> src_pos, src_mom;  // host copies of the dipoles (for H0 at receivers)
  bool contrast_set = false;
  int precond_kind = 0;  // ie_set_preconditioner: 0 none, 1 contraction IE
  // contraction-IE right preconditioner, built on first use: sym6 [6][N] each
  double* pre_p = nullptr;   // P = 2 sigma_b (sigma + sigma_b I)^-1
  double* pre_a = nullptr;   // a = P^-1
  double* pre_dp = nullptr;  // dsigma P
  char* ws = nullptr;
  size_t ws_bytes = 0;
  std::string err;
  long long launches = 0;
  // small pinned host staging for reductions / coefficients
  double2* h_red = nullptr;
  size_t h_red_cap = 0;
  double2* d_red = nullptr;  // device mirror for coefficient uploads
  bool gmres_device = false;  // Arnoldi recurrences on the device (IE_GMRES_DEVICE=1 at create)
  int* h_arnflag = nullptr;  // mapped pinned [m][S] step flags of the device-side Arnoldi
  int* d_arnflag = nullptr;  // its device alias
  size_t h_arn_cap = 0;
  std::vector<cudaEvent_t> ev_arn;  // one per Arnoldi step of a cycle (look-ahead)
  size_t d_red_cap = 0;
  // per-kernel profiling of the operator (ie_profile): events[i] brackets kernel kind[i]
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Mark {
    int kernel, ev0, ev1;  // kernel id 0..4 and the events bracketing one pass of it
  };
  std::vector<Mark> ev_marks;
  size_t ev_used = 0;
  // L2-resident slab pipeline of the y/z passes (operator.cu): three streams, ring events
  int* fused_cnt = nullptr;  // task / slot counters of the persistent fused operator kernels
  // K-D + K-E / K-A + K-B as one persistent kernel each (X1 through an L2 ring): opt-in with
  // IE_FUSED_DE=1 / IE_FUSED_AB=1 at create -- parity-tested, measured slower
  bool fused_de = false;
  bool fused_ab = false;
  bool slabs = false;
  bool aux_ready = false;
  cudaStream_t aux[3] = {};
  cudaEvent_t aux_ev[16] = {};
};

namespace ie {

// ------------------------------------------------------------------ status helpers
ie_status fail(ie_ctx* c, ie_status s, const std::string& msg);
ie_status cuda_fail(ie_ctx* c, cudaError_t e, const char* where);
#define IE_CUDA(ctx, call)                                           \
  do {                                                               \
    cudaError_t e__ = (call);                                        \
    if (e__ != cudaSuccess) return ie::cuda_fail((ctx), e__, #call); \
  } while (0)
#define IE_CHECK_LAUNCH(ctx, name)                                     \
  do {                                                                 \
    (ctx)->launches++;                                                 \
    cudaError_t e__ = cudaGetLastError();                              \
    if (e__ != cudaSuccess) return ie::cuda_fail((ctx), e__, (name)); \
  } while (0)

inline bool is_pow2(long long v) { return v >= 1 && (v & (v - 1)) == 0; }
inline int ilog2i(long long v) {
  int p = 0;
  while ((1LL << p) < v) ++p;
  return p;
}

// ----------------------------------------------------------------- entry points (internal)
// operator.cu
ie_status build_twiddles(ie_ctx* c);
ie_status launch_apply(ie_ctx* c, ApplyParams& p);  // p.items/n_items may exceed kMaxItems? no: caller splits
size_t apply_scratch_bytes(int nx, int ny, int nz, int n_items);
// green.cu
ie_status build_green(ie_ctx* c, int nx, int ny, int nz, GreenSpec* out);
// the spectra of a domain of (nx,ny,nz) cells starting at cell layer k0 (k0 only matters
// for layered backgrounds)
const GreenSpec* green_for(ie_ctx* c, int nx, int ny, int nz, int k0, ie_status* st);
cudaError_t fft_axis(int L, double2* data, long long inner, long long outer, const double2* tw, cudaStream_t s);
// layered.cu
ie_status build_layer_table(ie_ctx* c, const void* host_table);
ie_status build_layer_spec(ie_ctx* c, int nx, int ny, int nz, int k0, GreenSpec* out);
cudaError_t launch_zlayer(const ApplyParams& p, cudaStream_t s);
ie_status receivers_table(ie_ctx* c, const double2* e, int n_rx, const double2* e0rx, const cplx* h0, cplx* out,
                          double2* scratch, size_t scratch_elems);
double sigma_b_at(const ie_ctx* c, int k);  // background conductivity of cell layer k
// fields.cu
ie_status pack_contrast(ie_ctx* c, const void* sigma_dev, int layout);
ie_status compute_incident(ie_ctx* c, int n_src, const double* pos, const double* moment, double2* out);
ie_status receivers(ie_ctx* c, const double2* e, int n_rx, const double* rx, cplx* h_out, const double* src_pos,
                    const double* src_mom, int n_src, double2* scratch /* >= (296 + n_src*n_rx)*3 */);
void launch_gather(ie_ctx* c, const double2* full, double2* box, const ie_box& b, int nsys, long long full_stride,
                   long long box_stride);
void launch_scatter(ie_ctx* c, double2* full, const double2* box, const ie_box& b, int nsys, long long full_stride,
                    long long box_stride);
void launch_axpby(ie_ctx* c, double2* z, cplx a, const double2* x, cplx b, const double2* y, long long n);
ie_status ensure_precond(ie_ctx* c);
// y = M x per cell (M sym6 over the grid with strides (cs, zs, ys), x, y compact [3][bz][by][bx])
void launch_cellmat(ie_ctx* c, double2* y, const double2* x, const double* M, int bx, int by, int bz, long long cs,
                    long long zs, long long ys);
// sums of |a - b|^2 (b may be null) per system; result doubles on host
ie_status norms2(ie_ctx* c, const double2* a, const double2* b, int nsys, long long len, long long stride,
                 double* out_host);
// krylov.cu
struct GmresSystem {
  const double2* b;  // rhs (compact over the domain)
  double2* x;        // initial guess in, solution out
  const double* dsig;  // dsigma, or dsigma P when preconditioned
  double tol;
  int min_iters;
  const double* pm = nullptr;  // right preconditioner P = 2 sigma_b (sigma + sigma_b I)^-1 (sym6) or null
  const double* pa = nullptr;  // its inverse a = (sigma + sigma_b I) / (2 sigma_b): chi0 = a x0
};
struct GmresResult {
  int iters = 0, restarts = 0, converged = 0, breakdown = 0;
  double relres_est = 0, relres_true = 0;
};
ie_status gmres_batched(ie_ctx* c, Arena& ar, int nx, int ny, int nz, int k0, long long ds_zs, long long ds_ys,
                        const std::vector<GmresSystem>& sys, int restart, int max_iters,
                        std::vector<GmresResult>& res, long long* applies);
size_t gmres_scratch_bytes(int nx, int ny, int nz, int nsys, int restart);
// single full-length vectors (FGMRES outer basis): h_j = <V_j, w>, ||w||^2 (host results);
// out = base + sum_j coef_j V_j
ie_status vec_dots(ie_ctx* c, Arena& ar, const double2* w, const double2* V, int nv, long long len, cplx* h,
                   double* wn2);
ie_status vec_axpy(ie_ctx* c, Arena& ar, double2* out, const double2* base, const double2* V, int nv,
                   const cplx* coef, long long len);

}  // namespace ie
