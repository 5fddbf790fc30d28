// Restarted GMRES (Saad & Schultz 1986) batched over independent systems that
// share one operator shape (the right-hand sides of one domain, or the equal-shape
// sub-domains of a Jacobi sweep).  Device side: the operator (operator.cu), fused
// multi-vector dot products (w read once per 16 basis vectors), fused multi-axpy, fixed-order
// reductions.  Host side: Hessenberg / Givens recurrences (O(m^2) scalars per system).
//
// Orthogonalisation: classical Gram-Schmidt with the DGKS re-orthogonalisation test
// (repeat once if ||w_after||^2 < eta2 ||w_before||^2, using ||w_after||^2 = ||w||^2 -
// sum |h_j|^2; eta2 below); the basis is kept unnormalised with a per-vector scale 1/beta that the next
// operator application folds into its load (ApplyItem::xscale).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "fft_core.cuh"
#include "ie_internal.h"
#include "pdl.cuh"

namespace ie {

constexpr int kDotG = 8;  // basis vectors per pass over w (one CTA group each)

struct DotJob {
  const double2* w;
  const double2* V;  // first basis vector; vector j at V + j * len
  int nv;            // number of basis vectors (dots); row nv gets ||w||^2 in .x
  int row;           // output row base
  const int* enable = nullptr;  // device flag: the job is skipped when *enable == 0 (null: always run)
};
struct AxpyJob {
  double2* out;
  const double2* base;  // may be null (then 0)
  const double2* V;
  int nv;
  int coef;  // offset into the coefficient array
  const int* enable = nullptr;
};

__device__ __forceinline__ double2 shfl_down2(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

// Dot products of w with G consecutive basis vectors (and ||w||^2 when the group reaches
// row nv): blockIdx.y selects the group, blockIdx.z the job.  All G+1 loads of an element
// are issued before the FMAs (uniform predicates, no divergence) so each thread keeps
// (G+1) x 16 bytes in flight; two elements per thread per trip for more memory parallelism.
template <int G>
__device__ __forceinline__ void mdot_body(const DotJob& jb, long long len, double2* __restrict__ part, int nblk) {
  const int g0 = blockIdx.y * G;
  if (g0 > jb.nv) return;
  if (jb.enable && *jb.enable == 0) return;
  __shared__ double2 red[8][G];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2 acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = czero();
  const long long stride = (long long)nblk * 256;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < len; i += 2 * stride) {
    const long long i2 = i + stride;
    const bool ok2 = i2 < len;
    double2 w[2], v[2][G];
    w[0] = jb.w[i];
    w[1] = ok2 ? jb.w[i2] : czero();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const bool on = g0 + g < jb.nv;
      v[0][g] = on ? jb.V[(long long)(g0 + g) * len + i] : czero();
      v[1][g] = (on && ok2) ? jb.V[(long long)(g0 + g) * len + i2] : czero();
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (g0 + g < jb.nv) {
          acc[g].x = fma(v[e][g].x, w[e].x, fma(v[e][g].y, w[e].y, acc[g].x));  // conj(v) * w
          acc[g].y = fma(v[e][g].x, w[e].y, fma(-v[e][g].y, w[e].x, acc[g].y));
        } else if (g0 + g == jb.nv) {
          acc[g].x = fma(w[e].x, w[e].x, fma(w[e].y, w[e].y, acc[g].x));
        }
      }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc[g] = cadd(acc[g], shfl_down2(acc[g], d));
  }
  if (lane == 0)
#pragma unroll
    for (int g = 0; g < G; ++g) red[wid][g] = acc[g];
  __syncthreads();
  if (threadIdx.x < G) {
    const int j = g0 + threadIdx.x;
    double2 sum = czero();
    for (int w8 = 0; w8 < 8; ++w8) sum = cadd(sum, red[w8][threadIdx.x]);
    if (j <= jb.nv) part[(long long)(jb.row + j) * nblk + blockIdx.x] = sum;
  }
}

template <int G>
__global__ void __launch_bounds__(256) k_mdot(const DotJob* __restrict__ jobs, long long len, double2* __restrict__ part,
                                              int nblk) {
  mdot_body<G>(jobs[blockIdx.z], len, part, nblk);
}

// the same with the jobs passed by value (no job upload before the launch, so the multi-dot
// follows the operator's last pass in the programmatic-dependent-launch chain, pdl.cuh)
constexpr int kMaxDotJobs = 64;
struct DotJobs {
  DotJob j[kMaxDotJobs];
};
template <int G>
__global__ void __launch_bounds__(256) k_mdot_val(const __grid_constant__ DotJobs jobs, long long len,
                                                  double2* __restrict__ part, int nblk) {
  pdl_wait();
  mdot_body<G>(jobs.j[blockIdx.z], len, part, nblk);
  pdl_trigger_late();
}

__global__ void k_reduce_rows(const double2* __restrict__ part, int nblk, double2* __restrict__ out) {
  pdl_wait();
  const int row = blockIdx.x;
  __shared__ double2 red[128];
  double2 s = czero();
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s = cadd(s, part[(long long)row * nblk + i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[row] = red[0];
  pdl_trigger_late();
}

// out = base + sum_j coef_j V_j.  Eight basis loads of an element are issued before their FMAs
// (uniform predicates) so each thread keeps 8 x 16 bytes in flight.
__device__ __forceinline__ void maxpy_body(const AxpyJob& jb, const double2* __restrict__ coefs, long long len) {
  constexpr int G = 8;
  if (jb.enable && *jb.enable == 0) return;
  __shared__ double2 cf[160];
  for (int j = threadIdx.x; j < jb.nv; j += blockDim.x) cf[j] = coefs[jb.coef + j];
  __syncthreads();
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < len; i += (long long)gridDim.x * 256) {
    double2 a0 = jb.base ? jb.base[i] : czero(), a1 = czero();
    for (int j0 = 0; j0 < jb.nv; j0 += G) {
      double2 v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = j0 + g < jb.nv ? jb.V[(long long)(j0 + g) * len + i] : czero();
#pragma unroll
      for (int g = 0; g < G; g += 2) {
        if (j0 + g < jb.nv) a0 = cadd(a0, cmul(cf[j0 + g], v[g]));
        if (j0 + g + 1 < jb.nv) a1 = cadd(a1, cmul(cf[j0 + g + 1], v[g + 1]));
      }
    }
    jb.out[i] = cadd(a0, a1);
  }
}
__global__ void __launch_bounds__(256) k_maxpy(const AxpyJob* __restrict__ jobs, const double2* __restrict__ coefs,
                                               long long len) {
  maxpy_body(jobs[blockIdx.y], coefs, len);
}
// the same with jobs and coefficients passed by value (no upload before the launch; pdl.cuh)
constexpr int kMaxAxpyJobs = 16, kMaxAxpyCoefs = 256;
struct AxpyPack {
  AxpyJob j[kMaxAxpyJobs];
  double2 cf[kMaxAxpyCoefs];
};
__global__ void __launch_bounds__(256) k_maxpy_val(const __grid_constant__ AxpyPack pk, long long len) {
  pdl_wait();
  maxpy_body(pk.j[blockIdx.y], pk.cf, len);
  pdl_trigger_late();
}

// ------------------------------------------------------- device-side Arnoldi recurrences
// The Hessenberg column, DGKS test, Givens rotations and stopping rule of one Arnoldi step run on
// the device (one CTA / thread per system), so a GMRES cycle is enqueued without a host round trip
// per step: the host reads each step's "still iterating" flags one step late (look-ahead 1; a
// finished system's extra step is skipped by every kernel but the operator) and reads the
// recurrences back at the end of the cycle.  Same formulas, same order as the host path.
struct ArnState {
  double2* H;     // [S][m][m+1] column-major per system: H[(s m + k)(m+1) + j]
  double2* cs;    // [S][m]
  double2* sn;    // [S][m]
  double2* g;     // [S][m+1]
  double* scale;  // [S][m+1] basis scales 1/beta
  double2* h;     // [S][m+1] current column
  double* beta2;  // [S]
  double* bnorm;  // [S]
  double* tol;    // [S]
  double* est;    // [S]
  int* flag;      // [S] 1 while the system iterates in the cycle
  int* reorth;    // [S] DGKS second pass requested
  int* kdone;     // [S] Arnoldi steps done in the cycle
  int* iters;     // [S] total iterations
  int* miniters;  // [S]
  int* brk;       // [S] breakdown (non-finite)
  int m, maxiters;
};

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// Per-step jobs of the live systems, passed by value (no per-step job upload): system s's basis
// is V + s * sys_stride, w = V_{k+1}; its reduction rows and coefficients start at s * (m + 2).
struct ArnJobs {
  double2* V;
  long long sys_stride, len;
  int k, nlive;
  const int* enable;  // per-system flag array (flag or reorth)
  int ids[kMaxItems];
};

// multi-dot <V_j, w> (j <= k) and ||w||^2 of the live systems (k_mdot's body, jobs by value)
template <int G>
__global__ void __launch_bounds__(256) k_mdot_arn(const __grid_constant__ ArnJobs jb, double2* __restrict__ part,
                                                  int nblk, int st2) {
  const int s = jb.ids[blockIdx.z];
  const int nv = jb.k + 1;
  const int g0 = blockIdx.y * G;
  if (g0 > nv || !jb.enable[s]) return;
  const long long len = jb.len;
  const double2* Vb = jb.V + s * jb.sys_stride;
  const double2* w = Vb + (long long)(jb.k + 1) * len;
  __shared__ double2 red[8][G];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2 acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = czero();
  const long long stride = (long long)nblk * 256;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < len; i += 2 * stride) {
    const long long i2 = i + stride;
    const bool ok2 = i2 < len;
    double2 wv[2], v[2][G];
    wv[0] = w[i];
    wv[1] = ok2 ? w[i2] : czero();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const bool on = g0 + g < nv;
      v[0][g] = on ? Vb[(long long)(g0 + g) * len + i] : czero();
      v[1][g] = (on && ok2) ? Vb[(long long)(g0 + g) * len + i2] : czero();
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (g0 + g < nv) {
          acc[g].x = fma(v[e][g].x, wv[e].x, fma(v[e][g].y, wv[e].y, acc[g].x));
          acc[g].y = fma(v[e][g].x, wv[e].y, fma(-v[e][g].y, wv[e].x, acc[g].y));
        } else if (g0 + g == nv) {
          acc[g].x = fma(wv[e].x, wv[e].x, fma(wv[e].y, wv[e].y, acc[g].x));
        }
      }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc[g] = cadd(acc[g], shfl_down2(acc[g], d));
  }
  if (lane == 0)
#pragma unroll
    for (int g = 0; g < G; ++g) red[wid][g] = acc[g];
  __syncthreads();
  if (threadIdx.x < G) {
    const int j = g0 + threadIdx.x;
    double2 sum = czero();
    for (int w8 = 0; w8 < 8; ++w8) sum = cadd(sum, red[w8][threadIdx.x]);
    if (j <= nv) part[((long long)s * st2 + j) * nblk + blockIdx.x] = sum;
  }
}

// V_{k+1} -= sum_j coef_j V_j for the live systems (k_maxpy's body, jobs by value)
__global__ void __launch_bounds__(256) k_maxpy_arn(const __grid_constant__ ArnJobs jb,
                                                   const double2* __restrict__ coefs, int st2) {
  constexpr int G = 8;
  const int s = jb.ids[blockIdx.y];
  if (!jb.enable[s]) return;
  const int nv = jb.k + 1;
  const long long len = jb.len;
  const double2* Vb = jb.V + s * jb.sys_stride;
  double2* out = jb.V + s * jb.sys_stride + (long long)(jb.k + 1) * len;
  __shared__ double2 cf[160];
  for (int j = threadIdx.x; j < nv; j += blockDim.x) cf[j] = coefs[(long long)s * st2 + j];
  __syncthreads();
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < len; i += (long long)gridDim.x * 256) {
    double2 a0 = out[i], a1 = czero();
    for (int j0 = 0; j0 < nv; j0 += G) {
      double2 v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = j0 + g < nv ? Vb[(long long)(j0 + g) * len + i] : czero();
#pragma unroll
      for (int g = 0; g < G; g += 2) {
        if (j0 + g < nv) a0 = cadd(a0, cmul(cf[j0 + g], v[g]));
        if (j0 + g + 1 < nv) a1 = cadd(a1, cmul(cf[j0 + g + 1], v[g + 1]));
      }
    }
    out[i] = cadd(a0, a1);
  }
}

// Reduce the step's rows (one warp per row, fixed order), then h_j = <V_j, w> scale_j, the
// multi-axpy coefficients -h_j scale_j, beta^2 = ||w||^2 - sum |h_j|^2 and (pass 0) the DGKS
// request; pass 1 (always launched) then runs the step's Givens update (thread 0), so a step
// without re-orthogonalisation costs no extra launch beyond the two skipped pass-1 kernels.
__device__ void arn_givens(ArnState& a, int s, int k) {
  const int m = a.m;
  a.iters[s] += 1;
  // (reorth stays set for the pass-1 axpy launched after this kernel; the next step's pass 0
  // rewrites it; a stopping system clears it: its V_{k+1} is never used)
  if (a.brk[s]) {
    a.flag[s] = 0;
    a.reorth[s] = 0;
    return;
  }
  const double beta = sqrt(fmax(a.beta2[s], 0.0));
  double2* Hk = a.H + ((long long)s * m + k) * (m + 1);
  double2* cs = a.cs + s * m;
  double2* sn = a.sn + s * m;
  double2* g = a.g + s * (m + 1);
  for (int j = 0; j <= k; ++j) Hk[j] = a.h[s * (m + 1) + j];
  Hk[k + 1] = make_double2(beta, 0.0);
  for (int j = 0; j < k; ++j) {  // previous rotations
    const double2 t = cadd(cmul(cs[j], Hk[j]), cmul(sn[j], Hk[j + 1]));
    Hk[j + 1] = csub(cmul(cconj(cs[j]), Hk[j + 1]), cmul(cconj(sn[j]), Hk[j]));
    Hk[j] = t;
  }
  const double2 aa = Hk[k], bb = Hk[k + 1];
  const double den = sqrt(cabs2(aa) + cabs2(bb));
  if (den == 0.0) {
    cs[k] = make_double2(1.0, 0.0);
    sn[k] = czero();
  } else {
    cs[k] = cconj(make_double2(aa.x / den, aa.y / den));
    sn[k] = cconj(make_double2(bb.x / den, bb.y / den));
  }
  Hk[k] = cadd(cmul(cs[k], aa), cmul(sn[k], bb));
  Hk[k + 1] = czero();
  const double2 gk = g[k], ns = cconj(sn[k]);
  g[k + 1] = make_double2(-(ns.x * gk.x - ns.y * gk.y), -(ns.x * gk.y + ns.y * gk.x));
  g[k] = cmul(cs[k], gk);
  a.kdone[s] = k + 1;
  const double est = sqrt(cabs2(g[k + 1])) / a.bnorm[s];
  a.est[s] = est;
  const bool happy = !(beta > 1e-14 * sqrt(cabs2(Hk[k])));
  if ((est <= a.tol[s] && a.iters[s] >= a.miniters[s]) || a.iters[s] >= a.maxiters || happy) {
    a.flag[s] = 0;
    a.reorth[s] = 0;
  } else {
    a.scale[s * (m + 1) + k + 1] = 1.0 / beta;
  }
}

__global__ void __launch_bounds__(256) k_arn_step(ArnState a, const __grid_constant__ ArnJobs jb,
                                                  const double2* __restrict__ part, int nblk,
                                                  double2* __restrict__ coef, int pass, double eta2, int st2,
                                                  int* __restrict__ host_flag) {
  const int s = jb.ids[blockIdx.x];
  const int m = a.m, k = jb.k;
  if (!a.flag[s]) return;
  const bool work = pass == 0 || a.reorth[s];
  __shared__ double2 rows[130];
  __shared__ double hred[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (work) {
    for (int j = wid; j <= k + 1; j += 8) {  // one warp per row, fixed order
      double2 v = czero();
      const double2* pr = part + ((long long)s * st2 + j) * nblk;
      for (int i = lane; i < nblk; i += 32) v = cadd(v, pr[i]);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) v = cadd(v, shfl_down2(v, d));
      if (lane == 0) rows[j] = v;
    }
    __syncthreads();
    double hs = 0.0;
    for (int j = threadIdx.x; j <= k; j += blockDim.x) {
      const double sc = a.scale[s * (m + 1) + j];
      const double2 r = rows[j];
      const double2 hj = make_double2(r.x * sc, r.y * sc);
      double2* hp = a.h + s * (m + 1) + j;
      *hp = pass == 0 ? hj : cadd(*hp, hj);
      hs += cabs2(hj);
      coef[(long long)s * st2 + j] = make_double2(-hj.x * sc, -hj.y * sc);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) hs += __shfl_down_sync(0xffffffffu, hs, d);
    if (lane == 0) hred[wid] = hs;
    __syncthreads();
    if (threadIdx.x == 0) {
      double hsum = 0.0;
      for (int w8 = 0; w8 < 8; ++w8) hsum += hred[w8];
      const double ww = rows[k + 1].x;
      a.beta2[s] = ww - hsum;
      if (!isfinite(ww) || !isfinite(hsum)) a.brk[s] = 1;
      else if (pass == 0) a.reorth[s] = (ww - hsum < eta2 * ww) ? 1 : 0;
    }
  }
  if (pass == 1 && threadIdx.x == 0) {
    __threadfence_block();
    arn_givens(a, s, k);
    host_flag[s] = a.flag[s];  // mapped pinned memory: the host reads it after the step's event
  }
}

// ------------------------------------------------------------------------ host
void* Arena::take(size_t bytes) {
  const size_t a = (used + 255) & ~(size_t)255;
  used = a + bytes;
  if (used > peak) peak = used;
  if (counting || used > cap) return nullptr;
  return base + a;
}

// DGKS threshold on squared norms: re-orthogonalise when ||w_after||^2 < eta2 ||w_before||^2.
// Default eta = 0.1 (eta2 = 0.01, a tunable like Belos' DGKS depTol) rather than the textbook
// 1/sqrt(2): for this near-identity operator ||w_after||/||w_before|| stays in ~[0.1, 0.7], so
// 1/sqrt(2) re-orthogonalised every step (CGS2, 4 basis reads per iteration) while eta = 0.1
// gives bit-for-bit the same iteration counts and residuals to 1e-18 on c5 and c2mod at tol
// 1e-6 and 1e-9 with 2 basis reads.  IE_DGKS_ETA2 overrides.
static double dgks_eta2() {
  static const double v = [] {
    const char* e = getenv("IE_DGKS_ETA2");
    return e ? atof(e) : 0.01;
  }();
  return v;
}

// Arnoldi recurrences on the host (default: one host round trip per Arnoldi step) or on the
// device (IE_GMRES_DEVICE=1 when the context is created: look-ahead 1, no per-step round trip).
// Measured on B200: the device path is 3-12% SLOWER per iteration (c2mod
// 0.112 vs 0.101 ms, c3h 0.253 vs 0.225, c4h 0.705 vs 0.666, c5 6.27 vs 6.14): the
// always-launched DGKS second pass (two grids of early-exiting CTAs) and the extra step kernel
// cost more than the ~20 us round trip they remove.  Kept parity-tested, opt-in.

// CTAs per system for the multi-dot kernel: ~2368 CTAs in total (16 per SM)
static int dot_blocks(int nsys) { return std::max(32, std::min(1184, 2368 / std::max(1, nsys))); }

size_t gmres_scratch_bytes(int nx, int ny, int nz, int nsys, int restart) {
  const size_t len = 3ull * nx * ny * nz;
  const int items = std::min(nsys, kMaxItems);
  const int nblk = dot_blocks(nsys);
  size_t b = 0;
  auto add = [&](size_t x) { b = ((b + 255) & ~(size_t)255) + x; };
  add((size_t)nsys * (restart + 1) * len * sizeof(double2));           // V
  add(apply_scratch_bytes(nx, ny, nz, items));                          // X1/X2
  add((size_t)nsys * (restart + 2) * nblk * sizeof(double2));           // partials
  add((size_t)nsys * (restart + 2) * sizeof(double2));                  // reduced rows
  add((size_t)nsys * (restart + 2) * sizeof(double2) + nsys * 64 * 2);  // jobs + coefficients
  // device-side Arnoldi: H, cs, sn, g, scale, h, 10 per-system scalars, coefficients, rows, jobs
  const size_t S = nsys, m = restart;
  add(S * m * (m + 1) * sizeof(double2));
  add(S * m * sizeof(double2));
  add(S * m * sizeof(double2));
  add(S * (m + 1) * sizeof(double2));
  add(S * (m + 1) * sizeof(double));
  add(S * (m + 1) * sizeof(double2));
  for (int i = 0; i < 10; ++i) add(S * sizeof(double));
  add(S * (m + 2) * sizeof(double2));
  add(4096);
  return b + 1024;
}

namespace {

struct SysState {
  std::vector<cplx> H;  // (m+1) x m, column-major: H[k*(m+1) + j]
  std::vector<cplx> cs, sn, g;
  std::vector<double> scale;
  double bnorm = 0, beta = 0;
  int k = 0;          // Arnoldi steps in the current cycle
  bool active = true;  // still being solved
  bool cycle = false;  // iterating in the current cycle
};

}  // namespace

ie_status gmres_batched(ie_ctx* c, Arena& ar, int nx, int ny, int nz, int k0, long long ds_zs, long long ds_ys,
                        const std::vector<GmresSystem>& sys, int m, int max_iters, std::vector<GmresResult>& res,
                        long long* applies) {
  const int S = (int)sys.size();
  res.assign(S, GmresResult());
  if (S == 0) return IE_OK;
  const long long N = (long long)nx * ny * nz, len = 3 * N;
  const int items = std::min(S, kMaxItems);
  const int nblk = dot_blocks(S);
  ie_status st;
  const GreenSpec* gs = green_for(c, nx, ny, nz, k0, &st);
  if (!gs) return st;
  // staging (host pinned + device mirror): [dot jobs S*64 | axpy jobs S*64 | coefs S*(m+2)*16]
  const size_t jobs_bytes = (size_t)S * 64 * 2 + (size_t)S * (m + 2) * sizeof(double2);
  double2* V = (double2*)ar.take((size_t)S * (m + 1) * len * sizeof(double2));
  double2* scratch = (double2*)ar.take(apply_scratch_bytes(nx, ny, nz, items));
  double2* part = (double2*)ar.take((size_t)S * (m + 2) * nblk * sizeof(double2));
  double2* rows = (double2*)ar.take((size_t)S * (m + 2) * sizeof(double2));
  char* dstage = (char*)ar.take(jobs_bytes);
  if (!V || !scratch || !part || !rows || !dstage)
    return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for GMRES (need " + std::to_string(ar.peak) +
                                             " bytes; see ie_workspace_query)");
  const size_t rows_bytes = (size_t)S * (m + 2) * sizeof(double2);
  const size_t hneed = rows_bytes + jobs_bytes + 256;
  if (c->h_red_cap < hneed) {
    if (c->h_red) cudaFreeHost(c->h_red);
    c->h_red = nullptr;
    IE_CUDA(c, cudaMallocHost(&c->h_red, hneed));
    c->h_red_cap = hneed;
  }
  char* hstage = (char*)c->h_red;
  double2* hrows = (double2*)hstage;  // results of reductions
  DotJob* h_dot = (DotJob*)(hstage + rows_bytes);
  AxpyJob* h_axpy = (AxpyJob*)(hstage + rows_bytes + (size_t)S * 64);
  double2* h_coef = (double2*)(hstage + rows_bytes + (size_t)S * 128);
  DotJob* d_dot = (DotJob*)dstage;
  AxpyJob* d_axpy = (AxpyJob*)(dstage + (size_t)S * 64);
  double2* d_coef = (double2*)(dstage + (size_t)S * 128);

  auto Vs = [&](int s, int j) { return V + ((long long)s * (m + 1) + j) * len; };

  ApplyParams ap{};
  ap.nx = nx;
  ap.ny = ny;
  ap.nz = nz;
  ap.ds_cs = (long long)c->g.nx * c->g.ny * c->g.nz;
  ap.ds_zs = ds_zs;
  ap.ds_ys = ds_ys;
  ap.ghat = gs->oct;
  ap.mhat = gs->mhat;
  ap.X1 = scratch;
  ap.X2 = scratch + (size_t)items * 3 * 2 * N;
  int devscale_k = -1;  // >= 0: the items' basis scale is read on the device (device-side Arnoldi)
  ArnState* anp = nullptr;
  // apply to a list of (system, input, output) with given coefficients
  auto apply = [&](const std::vector<int>& ids, std::vector<const double2*> xin, std::vector<double> xsc,
                   std::vector<double2*> yout, double alpha, double beta, int acc) -> ie_status {
    for (size_t b0 = 0; b0 < ids.size(); b0 += kMaxItems) {
      const int nb = (int)std::min<size_t>(kMaxItems, ids.size() - b0);
      ap.alpha = alpha;
      ap.beta = beta;
      ap.accumulate = acc;
      ap.n_items = nb;
      for (int i = 0; i < nb; ++i) {
        ApplyItem& it = ap.items[i];
        it.x = xin[b0 + i];
        it.y = yout[b0 + i];
        it.dsig = sys[ids[b0 + i]].dsig;
        it.pm = sys[ids[b0 + i]].pm;
        it.xscale = xsc[b0 + i];
        it.xscale_dev = (devscale_k >= 0 && anp) ? anp->scale + (size_t)ids[b0 + i] * (m + 1) + devscale_k : nullptr;
        it.sx0 = 0;
        it.sx1 = nx;
        it.sy0 = 0;
        it.sy1 = ny;
        it.sz0 = 0;
        it.sz1 = nz;
      }
      ie_status s2 = launch_apply(c, ap);
      if (s2) return s2;
      if (applies) *applies += nb;
    }
    return IE_OK;
  };
  // dots: for each id, rows [row_base + 0 .. nv] = <V_j, w> (j < nv), ||w||^2 ; returns on host
  auto dots = [&](const std::vector<int>& ids, const std::vector<const double2*>& w, const std::vector<int>& nv,
                  std::vector<int>& rowbase) -> ie_status {
    const int n = (int)ids.size();
    DotJob* hj = h_dot;
    int row = 0;
    rowbase.resize(n);
    for (int i = 0; i < n; ++i) {
      hj[i] = DotJob{w[i], Vs(ids[i], 0), nv[i], row};
      rowbase[i] = row;
      row += nv[i] + 1;
    }
    int maxnv = 0;
    for (int i = 0; i < n; ++i) maxnv = std::max(maxnv, nv[i]);
    if (n <= kMaxDotJobs) {
      DotJobs dj;
      for (int i = 0; i < n; ++i) dj.j[i] = hj[i];
      launch_pass(use_pdl(), k_mdot_val<kDotG>, dim3(nblk, maxnv / kDotG + 1, n), dim3(256), 0, c->stream, dj, len, part,
                  nblk);
    } else {
      IE_CUDA(c, cudaMemcpyAsync(d_dot, hj, n * sizeof(DotJob), cudaMemcpyHostToDevice, c->stream));
      k_mdot<kDotG><<<dim3(nblk, maxnv / kDotG + 1, n), 256, 0, c->stream>>>(d_dot, len, part, nblk);
    }
    IE_CHECK_LAUNCH(c, "k_mdot");
    launch_pass(use_pdl(), k_reduce_rows, dim3(row), dim3(128), 0, c->stream, (const double2*)part, nblk, rows);
    IE_CHECK_LAUNCH(c, "k_reduce_rows");
    IE_CUDA(c, cudaMemcpyAsync(hrows, rows, row * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
    IE_CUDA(c, cudaStreamSynchronize(c->stream));
    return IE_OK;
  };
  // axpy: out_i = base_i + sum_j coef_ij V_ij
  auto axpy = [&](const std::vector<AxpyJob>& jobs, const std::vector<cplx>& coefs) -> ie_status {
    const int n = (int)jobs.size();
    if (n == 0) return IE_OK;
    const int gx = (int)std::max<long long>(1, std::min<long long>((len + 255) / 256, 1184 / n + 1));
    if (n <= kMaxAxpyJobs && coefs.size() <= (size_t)kMaxAxpyCoefs) {
      AxpyPack pk;
      for (int i = 0; i < n; ++i) pk.j[i] = jobs[i];
      for (size_t i = 0; i < coefs.size(); ++i) pk.cf[i] = make_double2(coefs[i].real(), coefs[i].imag());
      launch_pass(use_pdl(), k_maxpy_val, dim3(gx, n), dim3(256), 0, c->stream, pk, len);
      IE_CHECK_LAUNCH(c, "k_maxpy");
      return IE_OK;
    }
    for (int i = 0; i < n; ++i) h_axpy[i] = jobs[i];
    for (size_t i = 0; i < coefs.size(); ++i) h_coef[i] = make_double2(coefs[i].real(), coefs[i].imag());
    IE_CUDA(c, cudaMemcpyAsync(d_axpy, h_axpy, n * sizeof(AxpyJob), cudaMemcpyHostToDevice, c->stream));
    IE_CUDA(c, cudaMemcpyAsync(d_coef, h_coef, coefs.size() * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
    k_maxpy<<<dim3(gx, n), 256, 0, c->stream>>>(d_axpy, d_coef, len);
    IE_CHECK_LAUNCH(c, "k_maxpy");
    return IE_OK;
  };

  // right preconditioning (contraction IE): iterate on chi = a x, return x = P chi
  for (int s = 0; s < S; ++s)
    if (sys[s].pa) launch_cellmat(c, sys[s].x, sys[s].x, sys[s].pa, nx, ny, nz, ap.ds_cs, ds_zs, ds_ys);

  std::vector<SysState> ss(S);
  for (auto& s : ss) {
    s.H.assign((size_t)(m + 1) * m, 0.0);
    s.cs.assign(m, 0.0);
    s.sn.assign(m, 0.0);
    s.g.assign(m + 1, 0.0);
    s.scale.assign(m + 1, 1.0);
  }
  // ||b||
  {
    std::vector<double> nb(S);
    for (int s = 0; s < S; ++s) {
      double v;
      st = norms2(c, sys[s].b, nullptr, 1, len, 0, &v);
      if (st) return st;
      nb[s] = sqrt(v);
      ss[s].bnorm = nb[s];
    }
  }
  // true residual r = b - A x into V[s][0]; beta, relres_true
  auto residual = [&](const std::vector<int>& ids) -> ie_status {
    std::vector<const double2*> xin;
    std::vector<double> xsc;
    std::vector<double2*> yo;
    for (int s : ids) {
      launch_axpby(c, Vs(s, 0), 1.0, sys[s].b, 0.0, nullptr, len);
      xin.push_back(sys[s].x);
      xsc.push_back(1.0);
      yo.push_back(Vs(s, 0));
    }
    ie_status s2 = apply(ids, xin, xsc, yo, -1.0, 1.0, 1);  // V0 = b - x + G dsigma x
    if (s2) return s2;
    for (int s : ids) {
      double v;
      s2 = norms2(c, Vs(s, 0), nullptr, 1, len, 0, &v);
      if (s2) return s2;
      ss[s].beta = sqrt(v);
      res[s].relres_true = ss[s].bnorm > 0 ? ss[s].beta / ss[s].bnorm : 0.0;
      if (!std::isfinite(v)) res[s].breakdown = 1;
    }
    return IE_OK;
  };
  std::vector<int> all;
  for (int s = 0; s < S; ++s) {
    if (ss[s].bnorm == 0.0) {  // b = 0 -> x = 0
      launch_axpby(c, sys[s].x, 0.0, sys[s].x, 0.0, nullptr, len);
      ss[s].active = false;
      res[s].converged = 1;
      continue;
    }
    all.push_back(s);
  }
  st = residual(all);
  if (st) return st;
  for (int s : all) {
    res[s].relres_est = res[s].relres_true;
    if (res[s].breakdown) ss[s].active = false;
    else if (res[s].relres_true <= sys[s].tol && sys[s].min_iters <= 0) {
      ss[s].active = false;
      res[s].converged = 1;
    } else if (max_iters <= 0) {
      ss[s].active = false;
    }
  }

  // ---- device-side Arnoldi (see k_arn_step); opt-in with IE_GMRES_DEVICE=1
  const bool dev = c->gmres_device && S <= kMaxItems;  // ArnJobs holds <= kMaxItems live systems
  ArnState an{};
  anp = &an;
  double2* d_coefs = nullptr;
  const int st2 = m + 2;
  if (dev) {
    auto takeA = [&](size_t bytes) { return ar.take(bytes); };
    an.H = (double2*)takeA((size_t)S * m * (m + 1) * sizeof(double2));
    an.cs = (double2*)takeA((size_t)S * m * sizeof(double2));
    an.sn = (double2*)takeA((size_t)S * m * sizeof(double2));
    an.g = (double2*)takeA((size_t)S * (m + 1) * sizeof(double2));
    an.scale = (double*)takeA((size_t)S * (m + 1) * sizeof(double));
    an.h = (double2*)takeA((size_t)S * (m + 1) * sizeof(double2));
    an.beta2 = (double*)takeA((size_t)S * sizeof(double));
    an.bnorm = (double*)takeA((size_t)S * sizeof(double));
    an.tol = (double*)takeA((size_t)S * sizeof(double));
    an.est = (double*)takeA((size_t)S * sizeof(double));
    an.flag = (int*)takeA((size_t)S * sizeof(int));
    an.reorth = (int*)takeA((size_t)S * sizeof(int));
    an.kdone = (int*)takeA((size_t)S * sizeof(int));
    an.iters = (int*)takeA((size_t)S * sizeof(int));
    an.miniters = (int*)takeA((size_t)S * sizeof(int));
    an.brk = (int*)takeA((size_t)S * sizeof(int));
    an.m = m;
    an.maxiters = max_iters;
    d_coefs = (double2*)takeA((size_t)S * st2 * sizeof(double2));
    if (!an.H || !an.brk || !d_coefs)
      return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for GMRES (need " + std::to_string(ar.peak) +
                                               " bytes; see ie_workspace_query)");
    const size_t hbytes = (size_t)m * S * sizeof(int) + 256;
    if (c->h_arn_cap < hbytes) {
      if (c->h_arnflag) cudaFreeHost(c->h_arnflag);
      c->h_arnflag = nullptr;
      IE_CUDA(c, cudaHostAlloc((void**)&c->h_arnflag, hbytes, cudaHostAllocMapped));
      IE_CUDA(c, cudaHostGetDevicePointer((void**)&c->d_arnflag, c->h_arnflag, 0));
      c->h_arn_cap = hbytes;
    }
    if (c->ev_arn.size() < (size_t)m) {
      while (c->ev_arn.size() < (size_t)m) {
        cudaEvent_t ev;
        IE_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->ev_arn.push_back(ev);
      }
    }
    std::vector<double> tolv(S), bn(S);
    std::vector<int> mi(S);
    for (int s2 = 0; s2 < S; ++s2) {
      tolv[s2] = sys[s2].tol;
      bn[s2] = ss[s2].bnorm;
      mi[s2] = sys[s2].min_iters;
    }
    IE_CUDA(c, cudaMemcpyAsync(an.tol, tolv.data(), S * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    IE_CUDA(c, cudaMemcpyAsync(an.bnorm, bn.data(), S * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    IE_CUDA(c, cudaMemcpyAsync(an.miniters, mi.data(), S * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    IE_CUDA(c, cudaMemsetAsync(an.brk, 0, S * sizeof(int), c->stream));
    IE_CUDA(c, cudaStreamSynchronize(c->stream));  // the host vectors above go out of scope
  }
  // one GMRES cycle with the recurrences on the device for the systems `act`
  auto device_cycle = [&](const std::vector<int>& act) -> ie_status {
    const int n = (int)act.size();
    {  // cycle start: scale_0 = 1/beta, g = (beta, 0, ...), flag = 1, kdone = 0, iters = host count
      std::vector<double> sc0(S, 0.0);
      std::vector<double2> g0((size_t)S * (m + 1), make_double2(0.0, 0.0));
      std::vector<int> fl(S, 0), it0(S, 0);
      for (int s2 = 0; s2 < S; ++s2) it0[s2] = res[s2].iters;
      for (int s2 : act) {
        sc0[s2] = 1.0 / ss[s2].beta;
        g0[(size_t)s2 * (m + 1)] = make_double2(ss[s2].beta, 0.0);
        fl[s2] = 1;
      }
      IE_CUDA(c, cudaMemcpy2DAsync(an.scale, (m + 1) * sizeof(double), sc0.data(), sizeof(double), sizeof(double), S,
                                   cudaMemcpyHostToDevice, c->stream));
      IE_CUDA(c, cudaMemcpyAsync(an.g, g0.data(), g0.size() * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
      IE_CUDA(c, cudaMemcpyAsync(an.flag, fl.data(), S * sizeof(int), cudaMemcpyHostToDevice, c->stream));
      IE_CUDA(c, cudaMemcpyAsync(an.iters, it0.data(), S * sizeof(int), cudaMemcpyHostToDevice, c->stream));
      IE_CUDA(c, cudaMemsetAsync(an.kdone, 0, S * sizeof(int), c->stream));
      IE_CUDA(c, cudaMemsetAsync(an.reorth, 0, S * sizeof(int), c->stream));
      IE_CUDA(c, cudaStreamSynchronize(c->stream));  // the staging vectors go out of scope
    }
    int* hflags = c->h_arnflag;  // mapped pinned [m][S], written by k_arn_step
    int* hflags_dev = c->d_arnflag;
    for (size_t i = 0; i < (size_t)m * S; ++i) hflags[i] = 1;
    std::vector<int> live = act;
    for (int k = 0; k < m && !live.empty(); ++k) {
      // w = A v_k (basis scale read on the device)
      std::vector<const double2*> xin;
      std::vector<double> xsc;
      std::vector<double2*> yo;
      for (int s2 : live) {
        xin.push_back(Vs(s2, k));
        xsc.push_back(1.0);
        yo.push_back(Vs(s2, k + 1));
      }
      devscale_k = k;
      ie_status sa = apply(live, xin, xsc, yo, 1.0, -1.0, 0);
      devscale_k = -1;
      if (sa) return sa;
      const int nl = (int)live.size();
      ArnJobs jb{};
      jb.V = V;
      jb.sys_stride = (long long)(m + 1) * len;
      jb.len = len;
      jb.k = k;
      jb.nlive = nl;
      for (int i = 0; i < nl; ++i) jb.ids[i] = live[i];
      const int gx = (int)std::max<long long>(1, std::min<long long>((len + 255) / 256, 1184 / nl + 1));
      for (int pass = 0; pass < 2; ++pass) {
        jb.enable = pass == 0 ? an.flag : an.reorth;
        k_mdot_arn<kDotG><<<dim3(nblk, (k + 1) / kDotG + 1, nl), 256, 0, c->stream>>>(jb, part, nblk, st2);
        IE_CHECK_LAUNCH(c, "k_mdot_arn");
        k_arn_step<<<nl, 256, 0, c->stream>>>(an, jb, part, nblk, d_coefs, pass, dgks_eta2(), st2,
                                               hflags_dev + (size_t)k * S);
        IE_CHECK_LAUNCH(c, "k_arn_step");
        k_maxpy_arn<<<dim3(gx, nl), 256, 0, c->stream>>>(jb, d_coefs, st2);
        IE_CHECK_LAUNCH(c, "k_maxpy_arn");
      }
      IE_CUDA(c, cudaEventRecord(c->ev_arn[k], c->stream));
      if (k >= 1) {  // look-ahead 1: the flags of step k-1 decide step k+1
        IE_CUDA(c, cudaEventSynchronize(c->ev_arn[k - 1]));
        std::vector<int> nxt;
        for (int s2 : live)
          if (hflags[(size_t)(k - 1) * S + s2]) nxt.push_back(s2);
        live.swap(nxt);
      }
    }
    IE_CUDA(c, cudaStreamSynchronize(c->stream));
    // the cycle's recurrences back to the host (the end-of-cycle update below uses them)
    std::vector<double2> Hh((size_t)S * m * (m + 1)), gh((size_t)S * (m + 1));
    std::vector<double> sch((size_t)S * (m + 1)), esth(S);
    std::vector<int> kd(S), ith(S), bk(S);
    IE_CUDA(c, cudaMemcpy(Hh.data(), an.H, Hh.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(gh.data(), an.g, gh.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(sch.data(), an.scale, sch.size() * sizeof(double), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(esth.data(), an.est, S * sizeof(double), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(kd.data(), an.kdone, S * sizeof(int), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(ith.data(), an.iters, S * sizeof(int), cudaMemcpyDeviceToHost));
    IE_CUDA(c, cudaMemcpy(bk.data(), an.brk, S * sizeof(int), cudaMemcpyDeviceToHost));
    for (int s2 : act) {
      SysState& q = ss[s2];
      q.k = kd[s2];
      for (int kk = 0; kk < q.k; ++kk)
        for (int j = 0; j <= kk + 1; ++j) {
          const double2 v = Hh[((size_t)s2 * m + kk) * (m + 1) + j];
          q.H[(size_t)kk * (m + 1) + j] = cplx(v.x, v.y);
        }
      for (int j = 0; j <= q.k; ++j) q.g[j] = cplx(gh[(size_t)s2 * (m + 1) + j].x, gh[(size_t)s2 * (m + 1) + j].y);
      for (int j = 0; j < q.k; ++j) q.scale[j] = sch[(size_t)s2 * (m + 1) + j];
      res[s2].iters = ith[s2];
      if (q.k > 0) res[s2].relres_est = esth[s2];
      if (bk[s2]) {
        res[s2].breakdown = 1;
        q.active = false;
      }
      q.cycle = false;
    }
    return IE_OK;
  };

  while (true) {
    std::vector<int> act;
    for (int s = 0; s < S; ++s)
      if (ss[s].active) act.push_back(s);
    if (act.empty()) break;
    for (int s : act) {
      SysState& q = ss[s];
      q.scale[0] = 1.0 / q.beta;
      std::fill(q.g.begin(), q.g.end(), cplx(0.0));
      q.g[0] = q.beta;
      q.k = 0;
      q.cycle = true;
    }
    if (dev) {  // ---- device-side recurrences: no host round trip per Arnoldi step
      st = device_cycle(act);
      if (st) return st;
    }
    for (int k = 0; k < (dev ? 0 : m); ++k) {
      std::vector<int> it;
      for (int s : act)
        if (ss[s].cycle) it.push_back(s);
      if (it.empty()) break;
      // w = A v_k  -> V[s][k+1]
      std::vector<const double2*> xin;
      std::vector<double> xsc;
      std::vector<double2*> yo;
      for (int s : it) {
        xin.push_back(Vs(s, k));
        xsc.push_back(ss[s].scale[k]);
        yo.push_back(Vs(s, k + 1));
      }
      st = apply(it, xin, xsc, yo, 1.0, -1.0, 0);
      if (st) return st;
      std::vector<std::vector<cplx>> h(it.size(), std::vector<cplx>(k + 1, 0.0));
      std::vector<double> beta2(it.size());
      std::vector<int> todo(it.size());
      for (size_t i = 0; i < it.size(); ++i) todo[i] = (int)i;
      for (int pass = 0; pass < 2 && !todo.empty(); ++pass) {
        std::vector<int> ids;
        std::vector<const double2*> w;
        std::vector<int> nv, rb;
        for (int i : todo) {
          ids.push_back(it[i]);
          w.push_back(Vs(it[i], k + 1));
          nv.push_back(k + 1);
        }
        st = dots(ids, w, nv, rb);
        if (st) return st;
        std::vector<AxpyJob> jobs;
        std::vector<cplx> coefs;
        std::vector<int> again;
        for (size_t t = 0; t < todo.size(); ++t) {
          const int i = todo[t], s = it[i];
          const double2* r = hrows + rb[t];
          const double ww = r[k + 1].x;
          double hs = 0;
          jobs.push_back(AxpyJob{Vs(s, k + 1), Vs(s, k + 1), Vs(s, 0), k + 1, (int)coefs.size()});
          for (int j = 0; j <= k; ++j) {
            const cplx hj = cplx(r[j].x, r[j].y) * ss[s].scale[j];
            h[i][j] += hj;
            hs += std::norm(hj);
            coefs.push_back(-hj * ss[s].scale[j]);
          }
          beta2[i] = ww - hs;
          if (!std::isfinite(ww) || !std::isfinite(hs)) res[s].breakdown = 1;
          else if (pass == 0 && beta2[i] < dgks_eta2() * ww) again.push_back(i);  // DGKS: re-orthogonalise
        }
        st = axpy(jobs, coefs);
        if (st) return st;
        todo = again;
      }
      for (size_t i = 0; i < it.size(); ++i) {
        const int s = it[i];
        SysState& q = ss[s];
        GmresResult& rr = res[s];
        rr.iters++;
        if (rr.breakdown) {
          q.cycle = false;
          q.active = false;
          continue;
        }
        const double beta = sqrt(std::max(beta2[i], 0.0));
        cplx* Hk = &q.H[(size_t)k * (m + 1)];
        for (int j = 0; j <= k; ++j) Hk[j] = h[i][j];
        Hk[k + 1] = beta;
        for (int j = 0; j < k; ++j) {  // previous rotations
          const cplx t = q.cs[j] * Hk[j] + q.sn[j] * Hk[j + 1];
          Hk[j + 1] = -std::conj(q.sn[j]) * Hk[j] + std::conj(q.cs[j]) * Hk[j + 1];
          Hk[j] = t;
        }
        const cplx a = Hk[k], bb = Hk[k + 1];
        const double den = sqrt(std::norm(a) + std::norm(bb));
        if (den == 0.0) {
          q.cs[k] = 1.0;
          q.sn[k] = 0.0;
        } else {
          q.cs[k] = std::conj(a / den);
          q.sn[k] = std::conj(bb / den);
        }
        Hk[k] = q.cs[k] * a + q.sn[k] * bb;
        Hk[k + 1] = 0.0;
        q.g[k + 1] = -std::conj(q.sn[k]) * q.g[k];
        q.g[k] = q.cs[k] * q.g[k];
        q.k = k + 1;
        rr.relres_est = std::abs(q.g[k + 1]) / q.bnorm;
        const bool happy = !(beta > 1e-14 * std::abs(Hk[k]));
        if ((rr.relres_est <= sys[s].tol && rr.iters >= sys[s].min_iters) || rr.iters >= max_iters || happy)
          q.cycle = false;
        else
          q.scale[k + 1] = 1.0 / beta;
      }
    }
    // end of cycle: x += V y  (upper-triangular solve on host), then the true residual
    std::vector<AxpyJob> jobs;
    std::vector<cplx> coefs;
    std::vector<int> upd;
    for (int s : act) {
      SysState& q = ss[s];
      if (q.k == 0) continue;
      const int kk = q.k;
      std::vector<cplx> y(kk);
      for (int j = kk - 1; j >= 0; --j) {
        cplx t = q.g[j];
        for (int l = j + 1; l < kk; ++l) t -= q.H[(size_t)l * (m + 1) + j] * y[l];
        y[j] = t / q.H[(size_t)j * (m + 1) + j];
      }
      jobs.push_back(AxpyJob{sys[s].x, sys[s].x, Vs(s, 0), kk, (int)coefs.size()});
      for (int j = 0; j < kk; ++j) coefs.push_back(y[j] * q.scale[j]);
      upd.push_back(s);
    }
    st = axpy(jobs, coefs);
    if (st) return st;
    std::vector<int> live;
    for (int s : act)
      if (!res[s].breakdown) live.push_back(s);
    st = residual(live);
    if (st) return st;
    for (int s : act) {
      SysState& q = ss[s];
      GmresResult& rr = res[s];
      if (rr.breakdown) {
        q.active = false;
        continue;
      }
      if (rr.relres_true <= sys[s].tol && rr.iters >= sys[s].min_iters) {
        rr.converged = 1;
        q.active = false;
      } else if (rr.iters >= max_iters || q.beta == 0.0) {
        q.active = false;
        rr.converged = q.beta == 0.0;
      } else {
        rr.restarts++;
      }
    }
  }
  for (int s = 0; s < S; ++s)
    if (sys[s].pm) launch_cellmat(c, sys[s].x, sys[s].x, sys[s].pm, nx, ny, nz, ap.ds_cs, ds_zs, ds_ys);
  return IE_OK;
}

// --------------------------------------------------------------- single-vector helpers
// (the FGMRES outer iteration of the Krylov-accelerated DD, api.cu)
ie_status vec_dots(ie_ctx* c, Arena& ar, const double2* w, const double2* V, int nv, long long len, cplx* h,
                   double* wn2) {
  const int nblk = dot_blocks(1);
  const size_t mark = ar.used;
  double2* part = (double2*)ar.take((size_t)(nv + 1) * nblk * sizeof(double2));
  double2* rows = (double2*)ar.take((size_t)(nv + 1) * sizeof(double2));
  if (!part || !rows) {
    ar.used = mark;
    return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for the outer Krylov basis");
  }
  DotJobs jobs;
  jobs.j[0] = DotJob{w, V, nv, 0};
  launch_pass(use_pdl(), k_mdot_val<kDotG>, dim3(nblk, nv / kDotG + 1, 1), dim3(256), 0, c->stream, jobs, len, part, nblk);
  IE_CHECK_LAUNCH(c, "k_mdot");
  launch_pass(use_pdl(), k_reduce_rows, dim3(nv + 1), dim3(128), 0, c->stream, (const double2*)part, nblk, rows);
  IE_CHECK_LAUNCH(c, "k_reduce_rows");
  std::vector<double2> hr(nv + 1);
  IE_CUDA(c, cudaMemcpyAsync(hr.data(), rows, (nv + 1) * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  ar.used = mark;
  for (int j = 0; j < nv; ++j) h[j] = cplx(hr[j].x, hr[j].y);
  *wn2 = hr[nv].x;
  return IE_OK;
}

ie_status vec_axpy(ie_ctx* c, Arena& ar, double2* out, const double2* base, const double2* V, int nv,
                   const cplx* coef, long long len) {
  if (nv == 0) {
    if (out != base) launch_axpby(c, out, 1.0, base, 0.0, nullptr, len);
    return IE_OK;
  }
  const size_t mark = ar.used;
  AxpyJob* aj = (AxpyJob*)ar.take(sizeof(AxpyJob));
  double2* cf = (double2*)ar.take((size_t)nv * sizeof(double2));
  if (!aj || !cf) {
    ar.used = mark;
    return fail(c, IE_ERR_OUT_OF_MEMORY, "workspace too small for the outer Krylov basis");
  }
  const AxpyJob hj{out, base, V, nv, 0};
  std::vector<double2> hc(nv);
  for (int j = 0; j < nv; ++j) hc[j] = make_double2(coef[j].real(), coef[j].imag());
  IE_CUDA(c, cudaMemcpyAsync(aj, &hj, sizeof(AxpyJob), cudaMemcpyHostToDevice, c->stream));
  IE_CUDA(c, cudaMemcpyAsync(cf, hc.data(), nv * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  const int gx = (int)std::max<long long>(1, std::min<long long>((len + 255) / 256, 1184));
  k_maxpy<<<dim3(gx, 1), 256, 0, c->stream>>>(aj, cf, len);
  IE_CHECK_LAUNCH(c, "k_maxpy");
  IE_CUDA(c, cudaStreamSynchronize(c->stream));  // the staging is released below
  ar.used = mark;
  return IE_OK;
}

}  // namespace ie
