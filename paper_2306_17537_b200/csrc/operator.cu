// The FFT-accelerated IE operator  y = alpha x + beta G(dsigma x)   (Eq. 8 / Eq. 10,
// P:60-74) as five sm_100a kernels over a 2x zero-padded grid:
//   K-A k_xfwd : J = dsigma * x fused into the load, zero-pad x, length-2nx forward FFT
//   K-B k_yfwd : zero-pad y, length-2ny forward FFT (tiles of W consecutive kx)
//   K-C per (kx,ky) column: forward z FFT (upper half zero) -> 3x3 spectral multiply with
//       the packed Green spectrum -> inverse z FFT -> crop; written in place.
//       k_zconv_tm (2nz = 128, 256; the default): spectra parked in tensor memory, Green
//       planes staged through shared memory; k_zconv16 (radix 16, 2nz = 64 and the
//       IE_KC_VARIANT=0 / IE_KC128_VARIANT=0 baseline); k_zconv (generic lengths)
//   K-D k_yinv : inverse y FFT, keep the first ny rows
//   K-E k_xinv : inverse x FFT, keep the first nx, y = alpha*x + beta*conv (+ y)
// The 1/(8 nx ny nz) normalisation is folded into the packed spectrum (green.cu).
// See DESIGN.md §Kernels for the traffic model (1344 N + 96 (nx+1)(ny+1)(nz+1) bytes).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "bulk_copy.cuh"
#include "fft_core.cuh"
#include "pdl.cuh"
#include "ie_internal.h"

namespace ie {

__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }



// =====================================================================  K-A
template <int L>
__global__ void __launch_bounds__(128, 5) k_xfwd(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  pdl_trigger();
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V, R0 = P::radix(0, false), RL = P::radix(P::NST - 1, false);
  extern __shared__ double2 sm[];
  const ApplyItem& it = p.items[blockIdx.y];
  const int rows_cta = blockDim.x / T;
  const int lr = threadIdx.x / T, t = threadIdx.x % T;
  const int sbx = it.sx1 - it.sx0, sby = it.sy1 - it.sy0, sbz = it.sz1 - it.sz0;
  const int row = blockIdx.x * rows_cta + lr;
  const bool valid = row < sby * sbz;
  const int yy = valid ? it.sy0 + row % sby : 0;
  const int zz = valid ? it.sz0 + row / sby : 0;
  const long long sN = (long long)sbx * sby * sbz;
  const double2* xrow = it.x + ((long long)(zz - it.sz0) * sby + (yy - it.sy0)) * sbx - it.sx0;
  const double* srow = it.dsig + zz * p.ds_zs + yy * p.ds_ys;
  const double xs = item_xscale(it);

  // J for the thread's (non-zero) first-stage inputs, then one line FFT per component (a
  // thread holds 3 x V/2 values of J plus the V values of the line in flight)
  double2 J[3][V / 2];
#pragma unroll
  for (int u = 0; u < V / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0 / 2; ++r) {  // r >= R0/2 <=> x >= nx: zero padding
      const int x = t + u * T + r * (L / R0);
      double2 J0 = czero(), J1 = czero(), J2 = czero();
      if (valid && x >= it.sx0 && x < it.sx1) {
        const double2 e0 = cscale(ld2(xrow + x), xs);
        const double2 e1 = cscale(ld2(xrow + sN + x), xs);
        const double2 e2 = cscale(ld2(xrow + 2 * sN + x), xs);
        const double sxx = __ldg(srow + x), syy = __ldg(srow + p.ds_cs + x), szz = __ldg(srow + 2 * p.ds_cs + x);
        const double sxy = __ldg(srow + 3 * p.ds_cs + x), sxz = __ldg(srow + 4 * p.ds_cs + x),
                     syz = __ldg(srow + 5 * p.ds_cs + x);
        J0 = make_double2(sxx * e0.x + sxy * e1.x + sxz * e2.x, sxx * e0.y + sxy * e1.y + sxz * e2.y);
        J1 = make_double2(sxy * e0.x + syy * e1.x + syz * e2.x, sxy * e0.y + syy * e1.y + syz * e2.y);
        J2 = make_double2(sxz * e0.x + syz * e1.x + szz * e2.x, sxz * e0.y + syz * e1.y + szz * e2.y);
      }
      J[0][u * (R0 / 2) + r] = J0;
      J[1][u * (R0 / 2) + r] = J1;
      J[2][u * (R0 / 2) + r] = J2;
    }
  const int region = padded(L);
  auto idx = [&](int) { return SIdx{lr * region, 1, 0}; };
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double2 v[1][V];
#pragma unroll
    for (int u = 0; u < V / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) v[0][u * R0 + r] = r < R0 / 2 ? J[l][u * (R0 / 2) + r] : czero();
    fft_run<L, false, -1, 1, true>(v, sm, idx, t, p.tw_x, l > 0);
    if (valid) {
      double2* out = p.X1 + ((((long long)blockIdx.y * 3 + l) * p.nz + zz) * p.ny + yy) * L;
#pragma unroll
      for (int u = 0; u < V / RL; ++u)
#pragma unroll
        for (int r = 0; r < RL; ++r) out[t + u * T + r * (L / RL)] = v[0][u * RL + r];
    }
  }
  pdl_trigger_late();
}

// =====================================================================  K-B
template <int L>
__global__ void __launch_bounds__(512) k_yfwd(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  pdl_trigger();
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V, R0 = P::radix(0, false), RL = P::radix(P::NST - 1, false);
  extern __shared__ double2 sm[];
  const int W = blockDim.x / T;
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  // rev: the launch order runs from the last plane of every component down to the first, so
  // the first CTAs read the rows K-A wrote last (still in L2)
  int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  if (p.rev) {
    const int id = (int)(gridDim.x * gridDim.y * gridDim.z) - 1 -
                   (int)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
    bx = id % gridDim.x;
    const int rest = id / gridDim.x;
    bz = rest % gridDim.z;
    by = rest / gridDim.z;
  }
  const int item = bz / 3, q = bz % 3;
  const ApplyItem& it = p.items[item];
  const int Lx = 2 * p.nx, Xw = p.x2w;  // X2 row width: 2nx, or the slab width (slab pipeline)
  const int kx = p.k0x + bx * W + c;
  const int z = it.sz0 + by;
  const double2* src = p.X1 + (((long long)item * 3 + q) * p.nz + z) * p.ny * Lx + kx;
  double2 v[1][V];
#pragma unroll
  for (int u = 0; u < V / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int y = t + u * T + r * (L / R0);
      v[0][u * R0 + r] = (r < R0 / 2 && y >= it.sy0 && y < it.sy1) ? src[(long long)y * Lx] : czero();
    }
  auto idx = [&](int) { return SIdx{0, W, c}; };
  fft_run<L, false, -1, 1, true>(v, sm, idx, t, p.tw_y, false);
  double2* dst = p.X2 + (((long long)item * 3 + q) * p.nz + z) * (long long)L * Xw + (kx - p.k0x);
#pragma unroll
  for (int u = 0; u < V / RL; ++u)
#pragma unroll
    for (int r = 0; r < RL; ++r) dst[(long long)(t + u * T + r * (L / RL)) * Xw] = v[0][u * RL + r];
  pdl_trigger_late();
}

// =====================================================================  K-C
template <int L>
__global__ void __launch_bounds__(256) k_zconv(const __grid_constant__ ApplyParams p) {
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V;
  constexpr int R0 = P::radix(0, false), RF = P::radix(P::NST - 1, false);  // forward order F
  constexpr int RB0 = P::radix(0, true), RBL = P::radix(P::NST - 1, true);  // inverse in order B
  static_assert(RB0 == RF && RBL == R0, "order B reverses order F");
  extern __shared__ double2 sm[];
  const int W = blockDim.x / T;
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const int item = blockIdx.z;
  const ApplyItem& it = p.items[item];
  const int nx = p.nx, ny = p.ny, nz = p.nz, Lx = 2 * nx, Ly = 2 * ny;
  const int kx = blockIdx.x * W + c;
  // mirror pairs (ky, 2ny-ky) adjacent in launch order so their shared octant rows hit L2
  const int by = blockIdx.y;
  const int ky = (by == 0) ? 0 : (by == 1 ? ny : ((by & 1) ? Ly - (by >> 1) : (by >> 1)));
  const long long cs = (long long)nz * Ly * Lx;  // component stride
  double2* col = p.X2 + (long long)item * 3 * cs + (long long)ky * Lx + kx;
  const long long zs = (long long)Ly * Lx;

  // all (pruned) inputs of the 3 components first: 3*V/2 independent loads in flight
  double2 in[3][V / 2];
#pragma unroll
  for (int u = 0; u < V / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0 / 2; ++r) {  // r >= R0/2 <=> z >= nz: zero padding
      const int z = t + u * T + r * (L / R0);
      const bool ok = z >= it.sz0 && z < it.sz1;
#pragma unroll
      for (int l = 0; l < 3; ++l) in[l][u * (R0 / 2) + r] = ok ? col[l * cs + z * zs] : czero();
    }
  const int region = padded(L * W);
  // forward z-FFTs one component at a time (8 live values per thread); each spectrum is
  // parked in this thread's own slots of its region
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double2 v[1][V];
#pragma unroll
    for (int u = 0; u < V / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) v[0][u * R0 + r] = (r < R0 / 2) ? in[l][u * (R0 / 2) + r] : czero();
    auto idx = [&](int) { return SIdx{l * region, W, c}; };
    fft_run<L, false, -1, 1>(v, sm, idx, t, p.tw_z, false);
    if constexpr (P::NST > 1) __syncthreads();  // the last stage read other threads' slots
#pragma unroll
    for (int u = 0; u < V / RF; ++u)
#pragma unroll
      for (int r = 0; r < RF; ++r) sm[idx(0)(t + u * T + r * (L / RF))] = v[0][u * RF + r];
  }

  // spectral 3x3 multiply with the packed (octant) Green spectrum and parity signs, one kz
  // at a time on this thread's own slots
  const int ix = kx <= nx ? kx : Lx - kx;
  const int iy = ky <= ny ? ky : Ly - ky;
  const double sx = kx > nx ? -1.0 : 1.0, sy = ky > ny ? -1.0 : 1.0;
  const long long gcs = (long long)(nz + 1) * (ny + 1) * (nx + 1);
  const double2* g = p.ghat + (long long)iy * (nx + 1) + ix;
  const long long gzs = (long long)(ny + 1) * (nx + 1);
  auto sidx = [&](int l, int i) { return SIdx{l * region, W, c}(i); };
#pragma unroll 2
  for (int s = 0; s < V; ++s) {
    const int kz = t + (s / RF) * T + (s % RF) * (L / RF);
    const int iz = kz <= nz ? kz : L - kz;
    const double sz = kz > nz ? -1.0 : 1.0;
    const double2* gz = g + iz * gzs;
    const double2 gxx = ld2(gz), gyy = ld2(gz + gcs), gzz = ld2(gz + 2 * gcs);
    const double2 gxy = cscale(ld2(gz + 3 * gcs), sx * sy);
    const double2 gxz = cscale(ld2(gz + 4 * gcs), sx * sz);
    const double2 gyz = cscale(ld2(gz + 5 * gcs), sy * sz);
    const int i0 = sidx(0, kz), i1 = sidx(1, kz), i2 = sidx(2, kz);
    const double2 j0 = sm[i0], j1 = sm[i1], j2 = sm[i2];
    sm[i0] = cadd(cadd(cmul(gxx, j0), cmul(gxy, j1)), cmul(gxz, j2));
    sm[i1] = cadd(cadd(cmul(gxy, j0), cmul(gyy, j1)), cmul(gyz, j2));
    sm[i2] = cadd(cadd(cmul(gxz, j0), cmul(gyz, j1)), cmul(gzz, j2));
  }

  // inverse z-FFTs (order B starts on the positions order F ended on), crop to z < nz
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double2 v[1][V];
    auto idx = [&](int) { return SIdx{l * region, W, c}; };
#pragma unroll
    for (int u = 0; u < V / RF; ++u)
#pragma unroll
      for (int r = 0; r < RF; ++r) v[0][u * RF + r] = sm[idx(0)(t + u * T + r * (L / RF))];
    fft_run<L, true, +1, 1>(v, sm, idx, t, p.tw_zr, true);
#pragma unroll
    for (int u = 0; u < V / RBL; ++u)
#pragma unroll
      for (int r = 0; r < RBL / 2; ++r) {  // outputs z >= nz are discarded (crop)
        const int z = t + u * T + r * (L / RBL);
        col[l * cs + z * zs] = v[0][u * RBL + r];
      }
  }
}

// =====================================================================  K-C (radix 16)
// The same z-convolution for L = 2nz in {64, 128, 256} as two Stockham stages, radix 16
// then R1 = L/16 (inverse: R1 then 16), so each FFT crosses shared memory once.
//  * the tile (W consecutive kx at one ky, the nz non-zero rows of the 3 components,
//    W*16 B per row) is staged into shared memory by per-thread asynchronous copies
//    (LDGSTS), and the packed-Green rows the tile will need are prefetched into L2 at the
//    same time, so the spectral multiply later finds them on chip;
//  * T = L/16 threads per column, 16 values each; the first forward butterfly skips the
//    zero upper half, the last inverse butterfly produces only the kept lower half;
//  * the three spectra are parked in shared memory; the multiply walks the octant index iz
//    and serves the mirror pair kz = iz, L - iz from one read of the 6 Green components
//    (half the loads of a per-kz walk); the first batch of those loads is issued before
//    the last forward FFT, the second before the first batch is consumed;
//  * 128 threads and 100 KB per CTA: two CTAs per SM, so one CTA's copies and loads
//    overlap the other's arithmetic.
// Shared layout: element (i, c) of a region at R[i*W + c]; an 8-lane phase of a 128-bit
// access is 8 consecutive c, i.e. 128 contiguous bytes: conflict-free.
__device__ __forceinline__ double2 flip_if(double2 a, unsigned neg) {  // sign flip without FP64 ops
  return make_double2(__hiloint2double(__double2hiint(a.x) ^ (int)neg, __double2loint(a.x)),
                      __hiloint2double(__double2hiint(a.y) ^ (int)neg, __double2loint(a.y)));
}
// y = g0 j0 + g1 j1 + g2 j2 as fused chains (6 FP64 ops per real/imag part)
__device__ __forceinline__ double2 cdot3(double2 g0, double2 j0, double2 g1, double2 j1, double2 g2, double2 j2) {
  double re = -g2.y * j2.y;
  re = fma(g2.x, j2.x, re);
  re = fma(-g1.y, j1.y, re);
  re = fma(g1.x, j1.x, re);
  re = fma(-g0.y, j0.y, re);
  re = fma(g0.x, j0.x, re);
  double im = g2.y * j2.x;
  im = fma(g2.x, j2.y, im);
  im = fma(g1.y, j1.x, im);
  im = fma(g1.x, j1.y, im);
  im = fma(g0.y, j0.x, im);
  im = fma(g0.x, j0.y, im);
  return make_double2(re, im);
}

template <int L, int W>
__global__ void __launch_bounds__(128, 2) k_zconv16(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  constexpr int T = L / 16, R1 = L / 16, U = 16 / R1, NZ = L / 2;
  static_assert(L == 64 || L == 128 || L == 256, "radix-16 z-pass: L in {64,128,256}");
  extern __shared__ __align__(16) double2 sm[];
  double2* twl = sm + 3 * L * W;  // exp(-2 pi i m / L), m < L
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  // items fastest in launch order: the CTAs of one pencil tile for all right-hand sides run
  // together and share its Green rows through L2
  const int item = p.n_items == 1 ? 0 : blockIdx.x % p.n_items;
  const int xt = p.n_items == 1 ? blockIdx.x : blockIdx.x / p.n_items;
  const ApplyItem& it = p.items[item];
  const int nx = p.nx, ny = p.ny, Lx = 2 * nx, Ly = 2 * ny, Xw = p.x2w;
  const int kx0 = p.k0x + xt * W, kx = kx0 + c;
  const int by = blockIdx.y;  // mirror pairs (ky, 2ny-ky) adjacent in launch order (L2 reuse of G)
  const int ky = (by == 0) ? 0 : (by == 1 ? ny : ((by & 1) ? Ly - (by >> 1) : (by >> 1)));
  const long long cs = (long long)NZ * Ly * Xw, zs = (long long)Ly * Xw;
  double2* tile = p.X2 + (long long)item * 3 * cs + (long long)ky * Xw + (kx0 - p.k0x);
  const long long gcs = (long long)(NZ + 1) * (ny + 1) * (nx + 1);
  const long long gzs = (long long)(ny + 1) * (nx + 1);
  const int ix = kx <= nx ? kx : Lx - kx;
  const int iy = ky <= ny ? ky : Ly - ky;
  const double2* g = p.ghat + (long long)iy * (nx + 1) + ix;

  // ---- stage the non-zero rows z in [sz0, sz1) (zero the rest) and the twiddle powers;
  //      prefetch the Green rows (6 components x (nz+1) octant planes) into L2
  {
    const int z0 = it.sz0, z1 = it.sz1;
#pragma unroll
    for (int l = 0; l < 3; ++l)
      for (int z = t; z < NZ; z += T) {
        double2* d = &sm[(l * L + z) * W + c];
        if (z >= z0 && z < z1) cp_async16(d, tile + l * cs + z * zs + c);
        else *d = czero();
      }
    for (int m = threadIdx.x; m < L; m += blockDim.x) cp_async16(&twl[m], &p.pw_z[m]);
    const int ixmin = (kx0 + W - 1 <= nx) ? kx0 : Lx - kx0 - (W - 1);  // the tile's ix span (W | nx)
    const double2* g0 = p.ghat + (long long)iy * (nx + 1) + ixmin;
    for (int q = threadIdx.x; q < 6 * (NZ + 1); q += blockDim.x) {
      const double2* row = g0 + (q / (NZ + 1)) * gcs + (q % (NZ + 1)) * gzs;
      prefetch_l2(row);
      prefetch_l2(row + (W - 1));
    }
    cp_async_wait_all();
    __syncthreads();
  }

  // L = 256 (U = 1): forward stage-1 twiddles w^(r t) and inverse ones conj(w^(r t)) are the
  // same 15 values for every component -- keep them in registers
  double2 twr[L == 256 ? 16 : 1];
  if constexpr (L == 256) {
#pragma unroll
    for (int r = 1; r < 16; ++r) twr[r] = twl[r * t];
  }
  auto tw = [&](int r, int j) -> double2 {
    if constexpr (L == 256) return twr[r];
    else return twl[r * j];
  };

  // ---- forward z-FFT of component l in place; its spectrum (kz = j + 16 r) is parked in
  //      the thread's own slots
  auto forward = [&](int l) {
    double2* S = sm + l * L * W;
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = S[(t + r * T) * W + c];  // z = t + r L/16 < nz
    dft16<-1, true>(v);
    __syncthreads();  // all inputs of this component read before the exchange overwrites them
#pragma unroll
    for (int r = 0; r < 16; ++r) S[(t * 16 + r) * W + c] = v[r];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        double2 x = S[(j + r * 16) * W + c];
        if (r > 0) x = cmul(x, tw(r, j));
        v[u * R1 + r] = x;
      }
      dftR<R1, -1>(&v[u * R1]);
#pragma unroll
      for (int r = 0; r < R1; ++r) S[(j + r * 16) * W + c] = v[u * R1 + r];
    }
  };

  // ---- 3x3 spectral multiply: octant plane iz = t + q T serves kz = iz and kz = L - iz; the
  //      full spectrum is D G_oct D with D = diag(sx, sy, sz) the per-axis mirror signs
  constexpr int NQ = NZ / T;           // octant planes per thread (plus iz = nz on t = 0)
  constexpr int B = NQ >= 4 ? NQ / 2 : NQ;  // planes per batch of loads
  const unsigned fx = kx > nx ? 0x80000000u : 0u, fy = ky > ny ? 0x80000000u : 0u;
  double2* S0 = sm;
  double2* S1 = sm + L * W;
  double2* S2 = sm + 2 * L * W;
  auto load_batch = [&](double2(&G)[B][6], int q0) {
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int k = 0; k < 6; ++k) G[b][k] = ld2(g + (t + (q0 + b) * T) * gzs + k * gcs);
  };
  auto mult = [&](int kz, unsigned fz, const double2(&G)[6]) {
    const double2 gxy = flip_if(G[3], fx ^ fy), gxz = flip_if(G[4], fx ^ fz), gyz = flip_if(G[5], fy ^ fz);
    const int a = kz * W + c;
    const double2 j0 = S0[a], j1 = S1[a], j2 = S2[a];
    S0[a] = cdot3(G[0], j0, gxy, j1, gxz, j2);
    S1[a] = cdot3(gxy, j0, G[1], j1, gyz, j2);
    S2[a] = cdot3(gxz, j0, gyz, j1, G[2], j2);
  };
  auto mult_batch = [&](const double2(&G)[B][6], int q0) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int iz = t + (q0 + b) * T;
      mult(iz, 0u, G[b]);
      if (iz != 0) mult(L - iz, 0x80000000u, G[b]);
    }
  };

  forward(0);
  double2 Ga[B][6];
  load_batch(Ga, 0);  // in flight during the last two forward FFTs
  forward(1);
  forward(2);
  __syncthreads();
  if constexpr (2 * B == NQ) {
    double2 Gb[B][6];
    load_batch(Gb, B);
    mult_batch(Ga, 0);
    mult_batch(Gb, B);
  } else {
    mult_batch(Ga, 0);
  }
  if (t == 0) {  // iz = nz: kz = nz only (its own mirror)
    double2 G[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) G[k] = ld2(g + NZ * gzs + k * gcs);
    mult(NZ, 0u, G);
  }
  __syncthreads();

  // ---- inverse z-FFTs (radix R1 then 16), crop to z < nz, store
#pragma unroll 1
  for (int l = 0; l < 3; ++l) {
    double2* S = sm + l * L * W;
    double2 v[16];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
#pragma unroll
      for (int r = 0; r < R1; ++r) v[u * R1 + r] = S[(j + r * 16) * W + c];
      dftR<R1, +1>(&v[u * R1]);
    }
    __syncthreads();  // every thread has read its spectrum slots before the exchange
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
#pragma unroll
      for (int r = 0; r < R1; ++r) S[(j * R1 + r) * W + c] = v[u * R1 + r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double2 x = S[(t + r * T) * W + c];
      if (r > 0) x = cmulc(x, tw(r, t));  // exp(+2 pi i r t / L)
      v[r] = x;
    }
    dft16<+1, false, true>(v);
    double2* dst = tile + l * cs + c;
#pragma unroll
    for (int r = 0; r < 8; ++r) dst[(long long)(t + r * T) * zs] = v[r];  // z = t + r L/16 < nz
  }
  pdl_trigger_late();
}

// K-C, TMEM-parked z-pass for L = 2nz in {128, 256}: T = L/16 threads per pencil, W = 2048/L pencils per CTA (128 threads, one TMEM
// lane each).  Forward: radix 16 (first stage, half the inputs zero) then U = 16/R1 radix-R1
// stages per thread (R1 = L/16), after which thread t holds kz = j + 16 r for j = t + u T
// (u < U, r < R1): 16 values per component.  Components 0, 1 are parked in the thread's TMEM lane,
// component 2 stays in registers, the 3x3 multiply is thread-local with the Green planes staged
// through shared memory in 4 chunks of NZ/4 + 1 octant planes (chunk k serves the r whose octant
// plane iz = min(kz, L - kz) falls in it, for every u), and the inverse starts from registers.
// Stage twiddles w^(r j) = w^(4a j) w^(b j) (r = 4a + b) from two loaded powers.  Threads of
// mirror-partner pencil positions (t, T - t) share a warp.
// the e-th stage-2 index r (ascending) whose Green octant plane falls in chunk k of the TMEM
// z-pass (chunk_of below); R1 = L/16 radix, CH = L/8 planes per chunk
template <int L>
__host__ __device__ constexpr int chunk_r(int k, int e) {
  constexpr int R1 = L / 16, CH = L / 8;
  int n = 0;
  for (int r = 0; r < R1; ++r) {
    const int ck = r < R1 / 2 ? (16 * r) / CH : (16 * (R1 - 1 - r)) / CH;
    if (ck == k) {
      if (n == e) return r;
      ++n;
    }
  }
  return -1;
}
static_assert(chunk_r<256>(0, 3) == 15 && chunk_r<256>(3, 0) == 6 && chunk_r<128>(0, 1) == 7 && chunk_r<128>(2, 0) == 2,
              "chunk slot enumeration");

// dft16 / dftR with the inner twiddles folded into the butterflies (FMA = true) or not
template <bool FMA, int DIR, bool HI = false, bool HO = false>
__device__ __forceinline__ void dft16k(double2* v) {
  if constexpr (FMA) dft16f<DIR, HI, HO>(v);
  else dft16<DIR, HI, HO>(v);
}
template <bool FMA, int R, int DIR>
__device__ __forceinline__ void dftRk(double2* v) {
  if constexpr (R == 16) dft16k<FMA, DIR>(v);
  else dftR<R, DIR>(v);
}

template <int L, bool kHoistTw = true, bool kPairMul = true, bool kFmaDft = true>
__global__ void __launch_bounds__(128, 3) k_zconv_tm(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  pdl_trigger();
  constexpr int NZ = L / 2, T = L / 16, W = 2048 / L, R1 = L / 16, U = 16 / R1;
  constexpr int CH = NZ / 4, GR = CH + 1;  // Green chunk: planes [CH k, CH k + CH]
  static_assert(L == 128 || L == 256, "TMEM z-pass: L in {128, 256}");
  static_assert(W * T == 128 && U * R1 == 16, "one TMEM lane per thread, 16 values per component");
  static_assert(6 * GR * W <= 2 * NZ * W, "a Green chunk fits one half of the staging area");
  constexpr uint32_t kCols = 128;
  extern __shared__ __align__(16) double2 sm[];
  double2* twl = sm + 4 * NZ * W;  // exp(-2 pi i m / L), m < L
  uint32_t* tslot = reinterpret_cast<uint32_t*>(twl + L);
  const int c = threadIdx.x % W, q = threadIdx.x / W;
  // pencil position t of lane group q, with t and its mirror partner T - t in one warp
  int t;
  if constexpr (L == 256) t = (q & 1) ? (q == 1 ? 8 : 16 - (q >> 1)) : (q >> 1);
  else t = (int)((0x53627140u >> (4 * q)) & 7);  // q -> {0, 4, 1, 7, 2, 6, 3, 5}
  const int item = p.n_items == 1 ? 0 : blockIdx.x % p.n_items;
  const int xt = p.n_items == 1 ? blockIdx.x : blockIdx.x / p.n_items;
  const ApplyItem& it = p.items[item];
  const int nx = p.nx, ny = p.ny, Lx = 2 * nx, Ly = 2 * ny, Xw = p.x2w;
  const int kx0 = p.k0x + xt * W, kx = kx0 + c;
  const int by = blockIdx.y;
  const int ky = (by == 0) ? 0 : (by == 1 ? ny : ((by & 1) ? Ly - (by >> 1) : (by >> 1)));
  const long long cs = (long long)NZ * Ly * Xw, zs = (long long)Ly * Xw;
  double2* tile = p.X2 + (long long)item * 3 * cs + (long long)ky * Xw + (kx0 - p.k0x);
  const long long gcs = (long long)(NZ + 1) * (ny + 1) * (nx + 1);
  const long long gzs = (long long)(ny + 1) * (nx + 1);
  const int ix = kx <= nx ? kx : Lx - kx;
  const int iy = ky <= ny ? ky : Ly - ky;
  const double2* g = p.ghat + (long long)iy * (nx + 1) + ix;

  if (threadIdx.x < 32) tmem_alloc(tslot, kCols);
  {
    const int z0 = it.sz0, z1 = it.sz1;
#pragma unroll
    for (int l = 0; l < 3; ++l)
      for (int z = q; z < NZ; z += T) {
        double2* d = &sm[(l * NZ + z) * W + c];
        if (z >= z0 && z < z1) cp_async16(d, tile + l * cs + z * zs + c);
        else *d = czero();
      }
    {
      for (int m = threadIdx.x; m < L; m += blockDim.x) cp_async16(&twl[m], &p.pw_z[m]);
    }
    cp_async_wait_all();  // (no L2 prefetch of the Green rows: the chunk copies run a pass ahead)
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  const uint32_t taddr = *tslot + ((uint32_t)(32 * (threadIdx.x / 32)) << 16);

  auto xrow = [&](int l, int row) -> double2* {
    return row < NZ ? sm + (l * NZ + row) * W + c : sm + (3 * NZ + row - NZ) * W + c;
  };
  auto g_chunk = [&](int k, double2* R) {
    for (int row = q; row < GR; row += T) {
      const double2* src = g + (CH * k + row) * gzs;
#pragma unroll
      for (int comp = 0; comp < 6; ++comp) cp_async16(R + (comp * GR + row) * W + c, src + comp * gcs);
    }
    cp_async_commit();
  };
  double2* const RA = sm;               // staging blocks 0-1
  double2* const RB = sm + 2 * NZ * W;  // staging block 2 + spare
  // v[r] *= w^(r j) (CONJ: conj) for r = 1 .. n-1, from w^j and w^(4j)
  auto twiddle = [&](double2* v, int n, int j, auto conj_tag) {
    constexpr bool CONJ = decltype(conj_tag)::value;
    const double2 b1 = twl[j], a1 = twl[4 * j];
    const double2 b2 = cmul(b1, b1), b3 = cmul(b2, b1);
    const double2 a2 = cmul(a1, a1), a3 = cmul(a2, a1);
    const double2 bb[4] = {make_double2(1.0, 0.0), b1, b2, b3};
    const double2 aa[4] = {make_double2(1.0, 0.0), a1, a2, a3};
#pragma unroll
    for (int r = 1; r < 16; ++r) {
      if (r >= n) break;
      const int a = r >> 2, b = r & 3;
      const double2 w = (a == 0) ? bb[b] : (b == 0 ? aa[a] : cmul(aa[a], bb[b]));
      v[r] = CONJ ? cmulc(v[r], w) : cmul(v[r], w);
    }
  };
  // L = 256 (U = 1, j = t): the 15 stage twiddles w^(r t) are the same for the three forward and
  // (conjugated) the three inverse transforms -- generated once per direction and kept in registers
  constexpr bool HOIST = (L == 256) && kHoistTw;
  double2 twr[HOIST ? 16 : 1];
  auto make_tw = [&]() {
    if constexpr (HOIST) {
      const double2 b1 = twl[t], a1 = twl[4 * t];
      const double2 b2 = cmul(b1, b1), b3 = cmul(b2, b1);
      const double2 a2 = cmul(a1, a1), a3 = cmul(a2, a1);
      const double2 bb[4] = {make_double2(1.0, 0.0), b1, b2, b3};
      const double2 aa[4] = {make_double2(1.0, 0.0), a1, a2, a3};
#pragma unroll
      for (int r = 1; r < 16; ++r) {
        const int a = r >> 2, b = r & 3;
        twr[r] = (a == 0) ? bb[b] : (b == 0 ? aa[a] : cmul(aa[a], bb[b]));
      }
    }
  };
  auto forward = [&](int l, double2(&v)[16], bool hook) {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = sm[(l * NZ + t + r * T) * W + c];  // z = t + r T < nz
    dft16k<kFmaDft, -1, true>(v);
    __syncthreads();  // every input row of component l read before the exchange overwrites it
    if (hook) g_chunk(0, RA);  // blocks 0-1 are free once component 1 is done
    {  // rows t*16 .. t*16+15 lie on one side of NZ (a multiple of 16): one select per pass
      double2* wb = xrow(l, t * 16);
#pragma unroll
      for (int r = 0; r < 16; ++r) wb[r * W] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
      // rows j + 16 r: below NZ exactly for r < R1/2 (j < 16)
      const double2* lo = sm + (l * NZ + j) * W + c;
      const double2* hi = sm + (3 * NZ + j) * W + c - (long long)NZ * W;
#pragma unroll
      for (int r = 0; r < R1; ++r) v[u * R1 + r] = (r < R1 / 2 ? lo : hi)[16 * r * W];
      if constexpr (HOIST) {
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], twr[r]);
      } else {
        twiddle(&v[u * R1], R1, j, std::false_type{});
      }
      dftRk<kFmaDft, R1, -1>(&v[u * R1]);  // v[u R1 + r] = spectrum at kz = j + 16 r
    }
  };
  const unsigned fx = kx > nx ? 0x80000000u : 0u, fy = ky > ny ? 0x80000000u : 0u;
  // chunk serving stage-2 index r: iz = kz = j + 16 r (r < R1/2) or L - kz (r >= R1/2)
  auto chunk_of = [](int r) { return r < R1 / 2 ? (16 * r) / CH : (16 * (R1 - 1 - r)) / CH; };

  double2 v[16];
  make_tw();
#pragma unroll 1
  for (int l = 0; l < 2; ++l) {
    forward(l, v, false);
#pragma unroll
    for (int i = 0; i < 4; ++i) tmem_st4(taddr + 64 * l + 16 * i, &v[4 * i]);
  }
  tmem_wait_st();
  forward(2, v, true);
  __syncthreads();  // block 2 + spare read
  g_chunk(1, RB);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k == 0) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();  // chunk k landed (all threads' copies); chunk k-1 fully consumed
    if (k == 1) g_chunk(2, RA);
    if (k == 2) g_chunk(3, RB);
    const double2* R = (k & 1) ? RB : RA;
    if constexpr (kPairMul) {
      // the chunk's four slots in two pairs: both slots' Green loads and TMEM loads are issued
      // before one wait, so their latencies overlap
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        double2 G[2][6];
        uint32_t raw[2][8];
        int sl[2], jj[2];
        unsigned fzz[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * pr + h;
          const int r = U == 1 ? chunk_r<L>(k, e) : chunk_r<L>(k, e >> 1), u = U == 1 ? 0 : (e & 1);
          const int s = u * R1 + r, j = t + u * T;
          sl[h] = s;
          jj[h] = j;
          const double2* gr = r < R1 / 2 ? R + (j + 16 * r - CH * k) * W + c : R + (L - j - 16 * r - CH * k) * W + c;
#pragma unroll
          for (int q6 = 0; q6 < 6; ++q6) G[h][q6] = gr[q6 * GR * W];
          fzz[h] = (r < R1 / 2 || (r == R1 / 2 && j == 0)) ? 0u : 0x80000000u;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld4_raw(taddr + 4 * sl[h], raw[h]);
          tmem_ld4_raw(taddr + 64 + 4 * sl[h], raw[h] + 4);
        }
        tmem_wait_ld16(&raw[0][0]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 gxy = flip_if(G[h][3], fx ^ fy), gxz = flip_if(G[h][4], fx ^ fzz[h]),
                        gyz = flip_if(G[h][5], fy ^ fzz[h]);
          const double2 j0 = raw_to_z(raw[h]), j1 = raw_to_z(raw[h] + 4), j2 = v[sl[h]];
          tmem_st1(taddr + 4 * sl[h], cdot3(G[h][0], j0, gxy, j1, gxz, j2));
          tmem_st1(taddr + 64 + 4 * sl[h], cdot3(gxy, j0, G[h][1], j1, gyz, j2));
          v[sl[h]] = cdot3(gxz, j0, gyz, j1, G[h][2], j2);
        }
        (void)jj;
      }
      continue;
    }
#pragma unroll
    for (int r = 0; r < R1; ++r) {
      if (chunk_of(r) != k) continue;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = u * R1 + r;  // slot of kz = j + 16 r
        uint32_t raw[8];
        tmem_ld4_raw(taddr + 4 * s, raw);
        tmem_ld4_raw(taddr + 64 + 4 * s, raw + 4);
        tmem_wait_ld8(raw);
        // kz = j + 16 r < NZ for r < R1/2 (j < 16); otherwise iz = L - kz (kz = NZ: its own mirror)
        const int j = t + u * T;
        const double2* gr = r < R1 / 2 ? R + (j + 16 * r - CH * k) * W + c : R + (L - j - 16 * r - CH * k) * W + c;
        double2 G[6];
#pragma unroll
        for (int q6 = 0; q6 < 6; ++q6) G[q6] = gr[q6 * GR * W];
        const unsigned fz = (r < R1 / 2 || (r == R1 / 2 && j == 0)) ? 0u : 0x80000000u;
        const double2 gxy = flip_if(G[3], fx ^ fy), gxz = flip_if(G[4], fx ^ fz), gyz = flip_if(G[5], fy ^ fz);
        const double2 j0 = raw_to_z(raw), j1 = raw_to_z(raw + 4), j2 = v[s];
        tmem_st1(taddr + 4 * s, cdot3(G[0], j0, gxy, j1, gxz, j2));
        tmem_st1(taddr + 64 + 4 * s, cdot3(gxy, j0, G[1], j1, gyz, j2));
        v[s] = cdot3(gxz, j0, gyz, j1, G[2], j2);
      }
    }
  }
  tmem_wait_st();

  // inverse z-FFT from registers: radix R1 per j, exchange, twiddle + radix 16, crop, store
  auto inverse = [&](int l, double2(&v)[16], double2* B) {
#pragma unroll
    for (int u = 0; u < U; ++u) dftRk<kFmaDft, R1, +1>(&v[u * R1]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
#pragma unroll
      for (int r = 0; r < R1; ++r) B[(j * R1 + r) * W + c] = v[u * R1 + r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = B[(t + r * T) * W + c];
    if constexpr (HOIST) {
#pragma unroll
      for (int r = 1; r < 16; ++r) v[r] = cmulc(v[r], twr[r]);  // exp(+2 pi i r t / L)
    } else {
      twiddle(v, 16, t, std::true_type{});  // exp(+2 pi i r t / L)
    }
    dft16k<kFmaDft, +1, false, true>(v);
    double2* dst = tile + l * cs + c;
#pragma unroll
    for (int r = 0; r < 8; ++r) dst[(long long)(t + r * T) * zs] = v[r];  // z = t + r T < nz
  };
  make_tw();
  inverse(2, v, sm);
#pragma unroll 1
  for (int l = 0; l < 2; ++l) {
#pragma unroll
    for (int i = 0; i < 4; ++i) tmem_ld4(taddr + 64 * l + 16 * i, &v[4 * i]);
    inverse(l, v, l == 0 ? sm + 2 * NZ * W : sm);
  }
  tmem_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tmem_fence_after();
    tmem_dealloc(*tslot, kCols);
  }
  pdl_trigger_late();
}

// =====================================================================  K-D
template <int L>
__global__ void __launch_bounds__(512, 2) k_yinv(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  pdl_trigger();
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V, R0 = P::radix(0, false), RL = P::radix(P::NST - 1, false);
  extern __shared__ double2 sm[];
  const int W = blockDim.x / T;
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const int item = blockIdx.z / 3, q = blockIdx.z % 3;
  const int Lx = 2 * p.nx, Xw = p.x2w;
  const int kx = p.k0x + blockIdx.x * W + c;
  const int z = blockIdx.y;
  const double2* src = p.X2 + (((long long)item * 3 + q) * p.nz + z) * (long long)L * Xw + (kx - p.k0x);
  double2 v[1][V];
#pragma unroll
  for (int u = 0; u < V / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0; ++r) v[0][u * R0 + r] = src[(long long)(t + u * T + r * (L / R0)) * Xw];
  auto idx = [&](int) { return SIdx{0, W, c}; };
  fft_run<L, false, +1, 1, false, true>(v, sm, idx, t, p.tw_y, false);
  double2* dst = p.X1 + (((long long)item * 3 + q) * p.nz + z) * p.ny * Lx + kx;
#pragma unroll
  for (int u = 0; u < V / RL; ++u)
#pragma unroll
    for (int r = 0; r < RL / 2; ++r) dst[(long long)(t + u * T + r * (L / RL)) * Lx] = v[0][u * RL + r];
  pdl_trigger_late();
}

// =====================================================================  K-E
// One component per CTA row group (blockIdx.y = item*3 + component): the inverse x-FFT and
// the identity update never mix components, so a thread holds one line (8 values) and the
// kernel runs at high occupancy.
template <int L, bool PRE>
__global__ void __launch_bounds__(128) k_xinv(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  pdl_trigger();
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V, R0 = P::radix(0, false), RL = P::radix(P::NST - 1, false);
  extern __shared__ double2 sm[];
  // rev: reverse launch order (the first CTAs read the planes K-D wrote last, still in L2)
  int bx = blockIdx.x, by = blockIdx.y;
  if (p.rev) {
    const int id = (int)(gridDim.x * gridDim.y) - 1 - (int)(blockIdx.x + gridDim.x * blockIdx.y);
    bx = id % gridDim.x;
    by = id / gridDim.x;
  }
  const int item = by / 3, l = by % 3;
  const ApplyItem& it = p.items[item];
  const int rows_cta = blockDim.x / T;
  const int lr = threadIdx.x / T, t = threadIdx.x % T;
  const int nx = p.nx, ny = p.ny, nz = p.nz;
  const int row = bx * rows_cta + lr;
  const bool valid = row < ny * nz;
  const int yy = valid ? row % ny : 0, zz = valid ? row / ny : 0;
  const long long N = (long long)nx * ny * nz;
  double2 v[1][V];
  {
    const double2* src = p.X1 + ((((long long)item * 3 + l) * nz + zz) * ny + yy) * L;
#pragma unroll
    for (int u = 0; u < V / R0; ++u)
#pragma unroll
      for (int r = 0; r < R0; ++r) v[0][u * R0 + r] = valid ? src[t + u * T + r * (L / R0)] : czero();
  }
  const int region = padded(L);
  auto idx = [&](int) { return SIdx{lr * region, 1, 0}; };
  fft_run<L, false, +1, 1, false, true>(v, sm, idx, t, p.tw_x, false);
  if (!valid) return;
  const long long off = ((long long)zz * ny + yy) * nx;
  const double a = p.alpha * item_xscale(it), b = p.beta;
  double2* yrow = it.y + l * N + off;
  const double2* xrow = it.x + l * N + off;
  // contraction-IE right preconditioner: the identity term is (P x)_l (row l of sym6 P)
  const int pc0 = l == 0 ? 0 : (l == 1 ? 3 : 4), pc1 = l == 0 ? 3 : (l == 1 ? 1 : 5), pc2 = l == 0 ? 4 : (l == 1 ? 5 : 2);
  const double* prow = PRE ? it.pm + zz * p.ds_zs + yy * p.ds_ys : nullptr;
  const double2* x0row = it.x + off;
#pragma unroll
  for (int u = 0; u < V / RL; ++u)
#pragma unroll
    for (int r = 0; r < RL / 2; ++r) {  // x >= nx discarded (crop)
      const int x = t + u * T + r * (L / RL);
      double2 o = cscale(v[0][u * RL + r], b);
      if (a != 0.0) {
        double2 xi;
        if constexpr (PRE) {
          const double q0 = __ldg(prow + pc0 * p.ds_cs + x), q1 = __ldg(prow + pc1 * p.ds_cs + x),
                       q2 = __ldg(prow + pc2 * p.ds_cs + x);
          const double2 e0 = ld2(x0row + x), e1 = ld2(x0row + N + x), e2 = ld2(x0row + 2 * N + x);
          xi = make_double2(q0 * e0.x + q1 * e1.x + q2 * e2.x, q0 * e0.y + q1 * e1.y + q2 * e2.y);
        } else {
          xi = ld2(xrow + x);
        }
        o.x = fma(a, xi.x, o.x);
        o.y = fma(a, xi.y, o.y);
      }
      if (p.accumulate) o = cadd(o, yrow[x]);
      yrow[x] = o;
    }
  pdl_trigger_late();
}

// =====================================================================  K-DE (fused)
// K-D and K-E in ONE persistent launch, the X1 hand-off through a small ring of plane buffers
// that stays in L2 (so the 96N-byte X1 intermediate is neither written to nor read from HBM).
// Work = planes P = (item, component, z); per plane NYT "Y-tasks" (the inverse y-FFT of 8
// consecutive kx columns: X2 -> ring slot, rows y < ny) and NXT "X-tasks" (the inverse x-FFT
// of RX rows of the slot -> crop -> identity update into y, exactly k_xinv's epilogue).  Tasks
// are handed out in a fixed order by an atomic counter: group g = the Y-tasks of plane g, then
// the X-tasks of plane g - D (lag D), so an X-task waits only on Y-tasks handed out earlier
// (per-slot counter ydone), and a Y-task reusing a slot waits only on the X-tasks of the plane
// S planes back (xdone), handed out earlier too (S > D): every wait is on strictly earlier
// tasks, already held by running CTAs -> no deadlock for any residency.  Producer: stores
// (plain stores: L1 is write-through), barrier, __threadfence + atomicAdd by one thread (cumulative); consumer: ld.acquire spin by one thread,
// barrier, __threadfence, loads with ld.cg (the ring is rewritten within the launch, so no
// L1 / non-coherent path).
struct FusedSched {
  int* cnt;  // [0] task counter, [1, 1+S) ydone, [1+S, 1+2S) xdone (zeroed before the launch)
  int S, D, NP, NYT, NXT, RX;
  long long slot_elems;  // ny * 2nx
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const int* p, int target) {
  int ns = 32;
  while (ld_acquire_gpu(p) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns *= 2;
  }
}

template <int LY>
struct FusedShape {
  static constexpr int W = 8;                            // kx columns per Y-task
  static constexpr int NT = W * FftPlan<LY>::T;          // threads per CTA
};

template <int LY, int LX, bool PRE>
__global__ void __launch_bounds__(FusedShape<LY>::NT, 1024 / FusedShape<LY>::NT) k_yxinv(const __grid_constant__ ApplyParams p,
                                                             const FusedSched fs) {
  using PY = FftPlan<LY>;
  using PX = FftPlan<LX>;
  constexpr int W = FusedShape<LY>::W, NT = FusedShape<LY>::NT;
  constexpr int TY = PY::T, VY = PY::V, R0Y = PY::radix(0, false), RLY = PY::radix(PY::NST - 1, false);
  constexpr int TX = PX::T, VX = PX::V, R0X = PX::radix(0, false), RLX = PX::radix(PX::NST - 1, false);
  static_assert(NT % TX == 0, "whole x-lines per CTA");
  extern __shared__ double2 sm[];
  const int nx = p.nx, ny = p.ny, nz = p.nz, Lx = 2 * nx;
  const long long N = (long long)nx * ny * nz;
  const int G = fs.NYT + fs.NXT;
  const int D = fs.D, NP = fs.NP;
  const long long total = (long long)NP * G;
  int* ydone = fs.cnt + 1;
  int* xdone = fs.cnt + 1 + fs.S;
  __shared__ int s_next[2];
  if (threadIdx.x == 0) s_next[0] = atomicAdd(fs.cnt, 1);
  for (int iter = 0;; ++iter) {
    __syncthreads();  // s_next[iter & 1] written; the previous task's smem use is over
    const int task = s_next[iter & 1];
    if (task >= total) break;
    // the next task index is fetched now, its atomic latency hidden behind this task
    if (threadIdx.x == 0) s_next[(iter + 1) & 1] = atomicAdd(fs.cnt, 1);
    // decode the task order: D groups of Y only, NP - D groups of Y + X, D groups of X only
    bool isy;
    int plane, sub;
    const int a = D * fs.NYT, b = a + (NP - D) * G;
    if (task < a) {
      isy = true;
      plane = task / fs.NYT;
      sub = task % fs.NYT;
    } else if (task < b) {
      const int r = task - a, g = r / G, w = r % G;
      isy = w < fs.NYT;
      plane = isy ? D + g : g;
      sub = isy ? w : w - fs.NYT;
    } else {
      const int r = task - b;
      isy = false;
      plane = NP - D + r / fs.NXT;
      sub = r % fs.NXT;
    }
    const int slot = plane % fs.S, gen = plane / fs.S;
    double2* ring = p.X1 + (long long)slot * fs.slot_elems;
    const int item = plane / (3 * nz), q = (plane / nz) % 3, z = plane % nz;
    if (isy) {
      const int c = threadIdx.x % W, t = threadIdx.x / W;
      const int kx = sub * W + c;
      const double2* src = p.X2 + (((long long)item * 3 + q) * nz + z) * (long long)LY * Lx + kx;
      double2 v[1][VY];
#pragma unroll
      for (int u = 0; u < VY / R0Y; ++u)
#pragma unroll
        for (int r = 0; r < R0Y; ++r) v[0][u * R0Y + r] = src[(long long)(t + u * TY + r * (LY / R0Y)) * Lx];
      auto idx = [&](int) { return SIdx{0, W, c}; };
      fft_run<LY, false, +1, 1, false, true>(v, sm, idx, t, p.tw_y, false);
      // the slot is free once the X-tasks of the plane S back have read it
      if (gen > 0 && threadIdx.x == 0) spin_until(xdone + slot, fs.NXT * gen);
      __syncthreads();
      double2* dst = ring + kx;
#pragma unroll
      for (int u = 0; u < VY / RLY; ++u)
#pragma unroll
        for (int r = 0; r < RLY / 2; ++r) dst[(long long)(t + u * TY + r * (LY / RLY)) * Lx] = v[0][u * RLY + r];
      __syncthreads();  // every store of the CTA issued; thread 0's fence is cumulative
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ydone + slot, 1);
      }
    } else {
      if (threadIdx.x == 0) spin_until(ydone + slot, fs.NYT * (gen + 1));
      __syncthreads();
      const ApplyItem& it = p.items[item];
      const int l = q;
      const int lr = threadIdx.x / TX, t = threadIdx.x % TX;
      const int yy = sub * fs.RX + lr;
      const bool valid = yy < ny;
      double2 v[1][VX];
      {
        const double2* src = ring + (long long)(valid ? yy : 0) * Lx;
#pragma unroll
        for (int u = 0; u < VX / R0X; ++u)
#pragma unroll
          for (int r = 0; r < R0X; ++r) v[0][u * R0X + r] = valid ? __ldcg(src + t + u * TX + r * (LX / R0X)) : czero();
      }
      const int region = padded(LX);
      auto idx = [&](int) { return SIdx{lr * region, 1, 0}; };
      fft_run<LX, false, +1, 1, false, true>(v, sm, idx, t, p.tw_x, false);
      if (valid) {
        const int zz = z;
        const long long off = ((long long)zz * ny + yy) * nx;
        const double al = p.alpha * item_xscale(it), be = p.beta;
        double2* yrow = it.y + l * N + off;
        const double2* xrow = it.x + l * N + off;
        const int pc0 = l == 0 ? 0 : (l == 1 ? 3 : 4), pc1 = l == 0 ? 3 : (l == 1 ? 1 : 5),
                  pc2 = l == 0 ? 4 : (l == 1 ? 5 : 2);
        const double* prow = PRE ? it.pm + zz * p.ds_zs + yy * p.ds_ys : nullptr;
        const double2* x0row = it.x + off;
#pragma unroll
        for (int u = 0; u < VX / RLX; ++u)
#pragma unroll
          for (int r = 0; r < RLX / 2; ++r) {  // x >= nx discarded (crop)
            const int x = t + u * TX + r * (LX / RLX);
            double2 o = cscale(v[0][u * RLX + r], be);
            if (al != 0.0) {
              double2 xi;
              if constexpr (PRE) {
                const double q0 = __ldg(prow + pc0 * p.ds_cs + x), q1 = __ldg(prow + pc1 * p.ds_cs + x),
                             q2 = __ldg(prow + pc2 * p.ds_cs + x);
                const double2 e0 = ld2(x0row + x), e1 = ld2(x0row + N + x), e2 = ld2(x0row + 2 * N + x);
                xi = make_double2(q0 * e0.x + q1 * e1.x + q2 * e2.x, q0 * e0.y + q1 * e1.y + q2 * e2.y);
              } else {
                xi = ld2(xrow + x);
              }
              o.x = fma(al, xi.x, o.x);
              o.y = fma(al, xi.y, o.y);
            }
            if (p.accumulate) o = cadd(o, yrow[x]);
            yrow[x] = o;
          }
      }
      __syncthreads();  // every ring read of this task has returned
      if (threadIdx.x == 0) atomicAdd(xdone + slot, 1);
    }
  }
}

// =====================================================================  K-AB (fused)
// K-A and K-B in one persistent launch, the same scheme as K-DE: planes P = (item, z) of the
// source z-range; per plane NAT "A-tasks" (contrast J = dsigma x and the x-forward FFT of RA
// rows, all three components: exactly k_xfwd, into a ring slot [3][ny][2nx]) and NBT =
// 3 * 2nx/8 "B-tasks" (the y-forward FFT of 8 kx columns of one component: exactly k_yfwd,
// ring -> X2).  Order: A-tasks of plane g, then B-tasks of plane g - D.
template <int LX, int LY>
__global__ void __launch_bounds__(FusedShape<LY>::NT, 512 / FusedShape<LY>::NT) k_xyfwd(const __grid_constant__ ApplyParams p,
                                                                const FusedSched fs) {
  using PX = FftPlan<LX>;
  using PY = FftPlan<LY>;
  constexpr int W = FusedShape<LY>::W, NT = FusedShape<LY>::NT;
  constexpr int TX = PX::T, VX = PX::V, R0X = PX::radix(0, false), RLX = PX::radix(PX::NST - 1, false);
  constexpr int TY = PY::T, VY = PY::V, R0Y = PY::radix(0, false), RLY = PY::radix(PY::NST - 1, false);
  static_assert(NT % TX == 0, "whole x-lines per CTA");
  extern __shared__ double2 sm[];
  const int ny = p.ny, Lx = 2 * p.nx;
  const int G = fs.NYT + fs.NXT;  // NYT: A-tasks per plane, NXT: B-tasks per plane
  const int D = fs.D, NP = fs.NP;
  const long long total = (long long)NP * G;
  int* adone = fs.cnt + 1;
  int* bdone = fs.cnt + 1 + fs.S;
  const ApplyItem& it0 = p.items[0];
  const int sbz = it0.sz1 - it0.sz0;
  __shared__ int s_next[2];
  if (threadIdx.x == 0) s_next[0] = atomicAdd(fs.cnt, 1);
  for (int iter = 0;; ++iter) {
    __syncthreads();
    const int task = s_next[iter & 1];
    if (task >= total) break;
    if (threadIdx.x == 0) s_next[(iter + 1) & 1] = atomicAdd(fs.cnt, 1);
    bool isa;
    int plane, sub;
    const int a = D * fs.NYT, b = a + (NP - D) * G;
    if (task < a) {
      isa = true;
      plane = task / fs.NYT;
      sub = task % fs.NYT;
    } else if (task < b) {
      const int r = task - a, g = r / G, w = r % G;
      isa = w < fs.NYT;
      plane = isa ? D + g : g;
      sub = isa ? w : w - fs.NYT;
    } else {
      const int r = task - b;
      isa = false;
      plane = NP - D + r / fs.NXT;
      sub = r % fs.NXT;
    }
    const int slot = plane % fs.S, gen = plane / fs.S;
    double2* ring = p.X1 + (long long)slot * fs.slot_elems;  // [3][ny][2nx]
    const int item = plane / sbz, zz = it0.sz0 + plane % sbz;
    const ApplyItem& it = p.items[item];
    if (isa) {
      const int lr = threadIdx.x / TX, t = threadIdx.x % TX;
      const int sbx = it.sx1 - it.sx0, sby = it.sy1 - it.sy0;
      const int rowi = sub * fs.RX + lr;
      const bool valid = rowi < sby;
      const int yy = it.sy0 + (valid ? rowi : 0);
      const long long sN = (long long)sbx * sby * sbz;
      const double2* xrow = it.x + ((long long)(zz - it.sz0) * sby + (yy - it.sy0)) * sbx - it.sx0;
      const double* srow = it.dsig + zz * p.ds_zs + yy * p.ds_ys;
      const double xs = item_xscale(it);
      double2 J[3][VX / 2];
#pragma unroll
      for (int u = 0; u < VX / R0X; ++u)
#pragma unroll
        for (int r = 0; r < R0X / 2; ++r) {
          const int x = t + u * TX + r * (LX / R0X);
          double2 J0 = czero(), J1 = czero(), J2 = czero();
          if (valid && x >= it.sx0 && x < it.sx1) {
            const double2 e0 = cscale(ld2(xrow + x), xs);
            const double2 e1 = cscale(ld2(xrow + sN + x), xs);
            const double2 e2 = cscale(ld2(xrow + 2 * sN + x), xs);
            const double sxx = __ldg(srow + x), syy = __ldg(srow + p.ds_cs + x), szz = __ldg(srow + 2 * p.ds_cs + x);
            const double sxy = __ldg(srow + 3 * p.ds_cs + x), sxz = __ldg(srow + 4 * p.ds_cs + x),
                         syz = __ldg(srow + 5 * p.ds_cs + x);
            J0 = make_double2(sxx * e0.x + sxy * e1.x + sxz * e2.x, sxx * e0.y + sxy * e1.y + sxz * e2.y);
            J1 = make_double2(sxy * e0.x + syy * e1.x + syz * e2.x, sxy * e0.y + syy * e1.y + syz * e2.y);
            J2 = make_double2(sxz * e0.x + syz * e1.x + szz * e2.x, sxz * e0.y + syz * e1.y + szz * e2.y);
          }
          J[0][u * (R0X / 2) + r] = J0;
          J[1][u * (R0X / 2) + r] = J1;
          J[2][u * (R0X / 2) + r] = J2;
        }
      const int region = padded(LX);
      auto idx = [&](int) { return SIdx{lr * region, 1, 0}; };
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double2 v[1][VX];
#pragma unroll
        for (int u = 0; u < VX / R0X; ++u)
#pragma unroll
          for (int r = 0; r < R0X; ++r) v[0][u * R0X + r] = r < R0X / 2 ? J[l][u * (R0X / 2) + r] : czero();
        fft_run<LX, false, -1, 1, true>(v, sm, idx, t, p.tw_x, l > 0);
        if (l == 0) {  // the slot is free once the B-tasks of the plane S back have read it
          if (gen > 0 && threadIdx.x == 0) spin_until(bdone + slot, fs.NXT * gen);
          __syncthreads();
        }
        if (valid) {
          double2* out = ring + ((long long)l * ny + yy) * LX;
#pragma unroll
          for (int u = 0; u < VX / RLX; ++u)
#pragma unroll
            for (int r = 0; r < RLX; ++r) out[t + u * TX + r * (LX / RLX)] = v[0][u * RLX + r];
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(adone + slot, 1);
      }
    } else {
      if (threadIdx.x == 0) spin_until(adone + slot, fs.NYT * (gen + 1));
      __syncthreads();
      const int nkx = Lx / W;
      const int q = sub / nkx, kx = (sub % nkx) * W + threadIdx.x % W;
      const int c = threadIdx.x % W, t = threadIdx.x / W;
      const double2* src = ring + (long long)q * ny * Lx + kx;
      double2 v[1][VY];
#pragma unroll
      for (int u = 0; u < VY / R0Y; ++u)
#pragma unroll
        for (int r = 0; r < R0Y; ++r) {
          const int y = t + u * TY + r * (LY / R0Y);
          v[0][u * R0Y + r] = (r < R0Y / 2 && y >= it.sy0 && y < it.sy1) ? __ldcg(src + (long long)y * Lx) : czero();
        }
      auto idx = [&](int) { return SIdx{0, W, c}; };
      fft_run<LY, false, -1, 1, true>(v, sm, idx, t, p.tw_y, false);
      double2* dst = p.X2 + (((long long)item * 3 + q) * p.nz + zz) * (long long)LY * Lx + kx;
#pragma unroll
      for (int u = 0; u < VY / RLY; ++u)
#pragma unroll
        for (int r = 0; r < RLY; ++r) dst[(long long)(t + u * TY + r * (LY / RLY)) * Lx] = v[0][u * RLY + r];
      __syncthreads();  // every ring read of this task has returned
      if (threadIdx.x == 0) atomicAdd(bdone + slot, 1);
    }
  }
}

// =====================================================================  host side
// twiddle tables for every L = 2^p and both radix orders
template <int L>
static void fill_tw(std::vector<double2>& out, bool rev) {
  using P = FftPlan<L>;
  for (int s = 1; s < P::NST; ++s) {
    const int R = P::radix(s, rev), Ns = P::ns(s, rev);
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < Ns; ++k) {
        // exp(-2 pi i r k / (Ns R)), argument reduced exactly in integers, long double trig
        const long long m = (long long)r * k, M = (long long)Ns * R;
        const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)M;
        out.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
      }
  }
}

const double2* Twiddles::get(int L, int rev) const { return dev + off[ilog2i(L)][rev ? 1 : 0]; }
const double2* Twiddles::powers(int L) const { return dev + pw[ilog2i(L)]; }


ie_status build_twiddles(ie_ctx* c) {
  std::vector<double2> h;
  h.push_back(make_double2(1, 0));  // keep offsets of 1-stage plans valid
  auto add = [&](int p, auto fn) {
    for (int rev = 0; rev < 2; ++rev) {
      c->tw.off[p][rev] = (int)h.size();
      fn(h, rev != 0);
      h.push_back(make_double2(1, 0));
    }
  };
  add(1, fill_tw<2>);
  add(2, fill_tw<4>);
  add(3, fill_tw<8>);
  add(4, fill_tw<16>);
  add(5, fill_tw<32>);
  add(6, fill_tw<64>);
  add(7, fill_tw<128>);
  add(8, fill_tw<256>);
  add(9, fill_tw<512>);
  add(10, fill_tw<1024>);
  for (int p = 1; p <= kMaxLog2; ++p) {  // power tables exp(-2 pi i m / L), m < L
    const long long L = 1LL << p;
    c->tw.pw[p] = (int)h.size();
    for (long long m = 0; m < L; ++m) {
      const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)L;
      h.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
  }
  IE_CUDA(c, cudaMalloc(&c->tw.dev, h.size() * sizeof(double2)));
  IE_CUDA(c, cudaMemcpy(c->tw.dev, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  return IE_OK;
}

size_t apply_scratch_bytes(int nx, int ny, int nz, int n_items) {
  const size_t n = (size_t)nx * ny * nz;
  return (size_t)n_items * 3 * (2 * n + 4 * n) * sizeof(double2);
}

// launch configuration -----------------------------------------------------------
struct Cfg {
  dim3 grid, block;
  size_t smem;
};

template <int L>
static int threads_per_line() {
  return FftPlan<L>::T;
}

// opt in to > 48 KB dynamic shared memory (once per kernel instance and size)
// (separate contexts may be driven from different host threads: the cache is locked)
static cudaError_t prep(const void* kernel, size_t smem) {
  static std::unordered_map<const void*, size_t> done;
  static std::mutex mu;
  if (smem <= 48 * 1024) return cudaSuccess;
  std::lock_guard<std::mutex> lock(mu);
  auto f = done.find(kernel);
  if (f != done.end() && f->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[kernel] = smem;
  return e;
}

// IE_REV=0: K-B and K-E walk their tiles in launch order instead of reverse order (reverse: the
// first CTAs read what the previous pass wrote last, while it is still in L2)
static int rev_order() {
  static const int r = [] {
    const char* v = getenv("IE_REV");
    return v ? atoi(v) : 1;
  }();
  return r;
}


// x-passes: rows_cta rows of 3 lines; y-passes: W columns; z-pass: W columns of 3 lines
static int rows_per_cta(int T) { return T >= 128 ? 1 : 128 / T; }
static int y_width(int T, int Lx) {
  int W = 256 / T;
  if (W < 8) W = (512 / T < 8) ? 512 / T : 8;  // <= 512 threads per CTA
  if (W > Lx) W = Lx;
  return W;
}
static int z_width(int L, int T, int Lx) {
  int W = 8;
  while (W > 1 && (size_t)3 * padded(L * W) * sizeof(double2) > 112 * 1024) W /= 2;
  while (W * T < 128 && W * 2 <= Lx && (size_t)3 * padded(L * W * 2) * sizeof(double2) <= 112 * 1024) W *= 2;
  if (W > Lx) W = Lx;
  return W;
}

#define IE_DISPATCH_L(Lval, FN, ...)      \
  switch (Lval) {                         \
    case 2: FN<2>(__VA_ARGS__); break;     \
    case 4: FN<4>(__VA_ARGS__); break;     \
    case 8: FN<8>(__VA_ARGS__); break;     \
    case 16: FN<16>(__VA_ARGS__); break;   \
    case 32: FN<32>(__VA_ARGS__); break;   \
    case 64: FN<64>(__VA_ARGS__); break;   \
    case 128: FN<128>(__VA_ARGS__); break; \
    case 256: FN<256>(__VA_ARGS__); break; \
    case 512: FN<512>(__VA_ARGS__); break; \
    case 1024: FN<1024>(__VA_ARGS__); break; \
    default: return cudaErrorInvalidValue; \
  }

template <int L>
static cudaError_t go_xfwd(const ApplyParams& p, cudaStream_t s, int max_rows) {
  const int T = FftPlan<L>::T, rows = rows_per_cta(T);
  const size_t smem = (size_t)rows * padded(L) * sizeof(double2);
  cudaError_t e = prep((const void*)k_xfwd<L>, smem);
  if (e) return e;
  launch_pass(use_pdl(), k_xfwd<L>, dim3((max_rows + rows - 1) / rows, p.n_items), dim3(rows * T), smem, s, p);
  return cudaGetLastError();
}
template <int L>
static cudaError_t go_yfwd(const ApplyParams& p, cudaStream_t s, int max_planes) {
  const int T = FftPlan<L>::T, W = y_width(T, 2 * p.nx);
  const size_t smem = (size_t)padded(L * W) * sizeof(double2);
  cudaError_t e = prep((const void*)k_yfwd<L>, smem);
  if (e) return e;
  ApplyParams q = p;
  q.rev = rev_order();
  launch_pass(use_pdl(), k_yfwd<L>, dim3(p.x2w / W, max_planes, 3 * p.n_items), dim3(W * T), smem, s, q);
  return cudaGetLastError();
}
template <int L>
static cudaError_t go_zconv(const ApplyParams& p, cudaStream_t s) {
  const int T = FftPlan<L>::T, W = z_width(L, T, 2 * p.nx);
  const size_t smem = (size_t)3 * padded(L * W) * sizeof(double2);
  cudaError_t e = prep((const void*)k_zconv<L>, smem);
  if (e) return e;
  k_zconv<L><<<dim3(2 * p.nx / W, 2 * p.ny, p.n_items), W * T, smem, s>>>(p);
  return cudaGetLastError();
}
// radix-16 z-pass: W columns per CTA with W*T <= 128 and W >= 8 (128-byte rows); returns 0
// when the shape needs the generic kernel
static int zconv16_width(int L, int Lx) {
  if (L != 64 && L != 128 && L != 256) return 0;
  int W = 128 / (L / 16);
  while (W > 8 && W > Lx) W /= 2;
  return (W >= 8 && Lx % W == 0) ? W : 0;
}
template <int L, int W>
static cudaError_t go_zconv16_w(const ApplyParams& p, cudaStream_t s) {
  const size_t smem = (size_t)(3 * L * W + L) * sizeof(double2);
  cudaError_t e = prep((const void*)k_zconv16<L, W>, smem);
  if (e) return e;
  launch_pass(use_pdl(), k_zconv16<L, W>, dim3(p.n_items * (p.x2w / W), 2 * p.ny), dim3(W * (L / 16)), smem, s, p);
  return cudaGetLastError();
}
template <int L, bool HT, bool PM, bool FM>
static cudaError_t go_zconv_tm_h(const ApplyParams& p, cudaStream_t s) {
  constexpr int W = 2048 / L;
  const size_t smem = (size_t)(4 * (L / 2) * W + L + 1) * sizeof(double2);
  cudaError_t e = prep((const void*)k_zconv_tm<L, HT, PM, FM>, smem);
  if (e) return e;
  launch_pass(use_pdl(), k_zconv_tm<L, HT, PM, FM>, dim3(p.n_items * (p.x2w / W), 2 * p.ny), dim3(128), smem, s, p);
  return cudaGetLastError();
}
template <int L>
static cudaError_t go_zconv_tm(const ApplyParams& p, cudaStream_t s) {
  // A/B switches: IE_KC_HOIST=0: per-transform stage twiddles (L = 256)
  // instead of once per direction; IE_KC_PAIR (default on for L = 128 only): the spectral
  // multiply in slot pairs (one TMEM wait per pair); IE_KC_FMA=0: dft16 with separate
  // inner-twiddle products
  static const int sw = [] {
    auto get = [](const char* n, bool dflt) {
      const char* v = getenv(n);
      return v ? atoi(v) != 0 : dflt;
    };
    return (get("IE_KC_HOIST", true) ? 4 : 0) | (get("IE_KC_PAIR", L == 128) ? 2 : 0) | (get("IE_KC_FMA", true) ? 1 : 0);
  }();
  switch (sw) {
    case 7: return go_zconv_tm_h<L, true, true, true>(p, s);
    case 6: return go_zconv_tm_h<L, true, true, false>(p, s);
    case 5: return go_zconv_tm_h<L, true, false, true>(p, s);
    case 3: return go_zconv_tm_h<L, false, true, true>(p, s);
    default: return go_zconv_tm_h<L, false, false, false>(p, s);
  }
}
static cudaError_t go_zconv16(const ApplyParams& p, cudaStream_t s, int W) {
  const int L = 2 * p.nz;
  if (L == 256) {
    // IE_KC_VARIANT=0 selects the shared-memory-parked z-pass k_zconv16<256, 8> (1.79 ms on c5)
    // instead of the TMEM-parked k_zconv_tm<256> (1.34 ms); DESIGN.md section 6 has the steps
    // between them
    static const int kc = [] {
      const char* e = getenv("IE_KC_VARIANT");
      return e ? atoi(e) : 8;
    }();
    if (kc != 0) return go_zconv_tm<256>(p, s);
    return go_zconv16_w<256, 8>(p, s);
  }
  // 8-pencil tiles (128-byte rows): more, smaller CTAs per SM measured faster than 128-thread
  // tiles for L = 128 (c4h K-C 0.212 -> 0.202 ms)
  if (L == 128) {
    // IE_KC128_VARIANT: 1 = TMEM-parked spectra (k_zconv_tm<128>, c4h apply 0.396 -> 0.366 ms,
    // the default when the tile width divides 2nx), 0 = k_zconv16<128, 8>
    static const int kc128 = [] {
      const char* e = getenv("IE_KC128_VARIANT");
      return e ? atoi(e) : 1;
    }();
    if (kc128 == 1 && (p.x2w % 16) == 0) return go_zconv_tm<128>(p, s);
    return go_zconv16_w<128, 8>(p, s);
  }
  if (L == 64)
    return W == 32 ? go_zconv16_w<64, 32>(p, s) : (W == 16 ? go_zconv16_w<64, 16>(p, s) : go_zconv16_w<64, 8>(p, s));
  return cudaErrorInvalidValue;
}
template <int L>
static cudaError_t go_yinv(const ApplyParams& p, cudaStream_t s) {
  const int T = FftPlan<L>::T, W = y_width(T, 2 * p.nx);
  const size_t smem = (size_t)padded(L * W) * sizeof(double2);
  cudaError_t e = prep((const void*)k_yinv<L>, smem);
  if (e) return e;
  launch_pass(use_pdl(), k_yinv<L>, dim3(p.x2w / W, p.nz, 3 * p.n_items), dim3(W * T), smem, s, p);
  return cudaGetLastError();
}
template <int L, bool PRE>
static cudaError_t go_xinv_p(const ApplyParams& p, cudaStream_t s) {
  const int T = FftPlan<L>::T, rows = rows_per_cta(T);
  const size_t smem = (size_t)rows * padded(L) * sizeof(double2);
  cudaError_t e = prep((const void*)k_xinv<L, PRE>, smem);
  if (e) return e;
  ApplyParams q = p;
  q.rev = rev_order();
  launch_pass(use_pdl(), k_xinv<L, PRE>, dim3((p.ny * p.nz + rows - 1) / rows, 3 * p.n_items), dim3(rows * T), smem, s, q);
  return cudaGetLastError();
}
template <int L>
static cudaError_t go_xinv(const ApplyParams& p, cudaStream_t s) {
  // items of one launch are either all preconditioned (contraction IE) or none
  return p.items[0].pm ? go_xinv_p<L, true>(p, s) : go_xinv_p<L, false>(p, s);
}

// K-DE: persistent fused y-inverse + x-inverse (see the kernel); returns cudaErrorNotSupported
// when the shape has no instance (the caller then runs K-D and K-E)
// Lag D (planes) between a plane's producer and consumer tasks: more than the planes' worth
// of tasks the resident CTAs hold at once, so a consumer rarely finds its plane unfinished;
// ring slots S = D + 3 (a producer reusing a slot waits on the consumers S planes back).
constexpr int kFusedMaxSlots = 120;  // counters: [1 + 2 S] ints per fused kernel, 256 reserved each
static void fused_lag(int grid, int tasks_per_plane, int np, int* D, int* S) {
  const int d = (grid + tasks_per_plane - 1) / tasks_per_plane + 2;
  *S = std::max(1, std::min(std::min(np, d + 3), kFusedMaxSlots));
  *D = std::max(0, std::min(d, *S - 1));
}
template <int LY, int LX, bool PRE>
static cudaError_t go_yxinv_p(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  constexpr int NT = FusedShape<LY>::NT;
  constexpr int TX = FftPlan<LX>::T, RX = NT / TX;
  const size_t smem = (size_t)std::max(padded(LY * FusedShape<LY>::W), RX * padded(LX)) * sizeof(double2);
  const void* kern = (const void*)k_yxinv<LY, LX, PRE>;
  cudaError_t e = prep(kern, smem);
  if (e) return e;
  static int grid = 0;  // resident CTAs (per instance; the device is fixed for the process)
  if (!grid) {
    int dev = 0, sms = 0, per = 0;
    if ((e = cudaGetDevice(&dev)) || (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) ||
        (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, smem)))
      return e;
    grid = std::max(1, per) * sms;
  }
  if (!c->fused_cnt && (e = cudaMalloc(&c->fused_cnt, 512 * sizeof(int)))) return e;
  FusedSched fs;
  fs.cnt = c->fused_cnt;
  fs.NP = p.n_items * 3 * p.nz;
  fs.NYT = 2 * p.nx / FusedShape<LY>::W;
  fs.RX = RX;
  fs.NXT = (p.ny + RX - 1) / RX;
  fused_lag(grid, fs.NYT + fs.NXT, fs.NP, &fs.D, &fs.S);
  fs.slot_elems = (long long)p.ny * 2 * p.nx;
  if ((e = cudaMemsetAsync(c->fused_cnt, 0, (1 + 2 * fs.S) * sizeof(int), s))) return e;
  const long long total = (long long)fs.NP * (fs.NYT + fs.NXT);
  k_yxinv<LY, LX, PRE><<<(int)std::min<long long>(grid, total), NT, smem, s>>>(p, fs);
  return cudaGetLastError();
}
template <int LY, int LX>
static cudaError_t go_yxinv_l(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  return p.items[0].pm ? go_yxinv_p<LY, LX, true>(c, p, s) : go_yxinv_p<LY, LX, false>(c, p, s);
}
static cudaError_t go_yxinv(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  if (!c->fused_de || p.x2w != 2 * p.nx || p.k0x != 0) return cudaErrorNotSupported;
  const int LY = 2 * p.ny, LX = 2 * p.nx;
#define IE_FUSED_CASE(a, b) \
  if (LY == a && LX == b) return go_yxinv_l<a, b>(c, p, s);
  IE_FUSED_CASE(512, 512)
  IE_FUSED_CASE(256, 512)
  IE_FUSED_CASE(256, 256)
  IE_FUSED_CASE(128, 256)
  IE_FUSED_CASE(128, 128)
  IE_FUSED_CASE(64, 128)
  IE_FUSED_CASE(128, 64)
  IE_FUSED_CASE(64, 64)
#undef IE_FUSED_CASE
  return cudaErrorNotSupported;
}

// K-AB: persistent fused contrast + x-forward + y-forward (see the kernel)
template <int LX, int LY>
static cudaError_t go_xyfwd_l(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  constexpr int NT = FusedShape<LY>::NT;
  constexpr int TX = FftPlan<LX>::T, RA = NT / TX;
  const size_t smem = (size_t)std::max(padded(LY * FusedShape<LY>::W), RA * padded(LX)) * sizeof(double2);
  const void* kern = (const void*)k_xyfwd<LX, LY>;
  cudaError_t e = prep(kern, smem);
  if (e) return e;
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, per = 0;
    if ((e = cudaGetDevice(&dev)) || (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) ||
        (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, smem)))
      return e;
    grid = std::max(1, per) * sms;
  }
  if (!c->fused_cnt && (e = cudaMalloc(&c->fused_cnt, 512 * sizeof(int)))) return e;
  const ApplyItem& it = p.items[0];
  FusedSched fs;
  fs.cnt = c->fused_cnt + 256;  // its own counters (K-DE uses [0, 256))
  fs.NP = p.n_items * (it.sz1 - it.sz0);
  fs.RX = RA;
  fs.NYT = (it.sy1 - it.sy0 + RA - 1) / RA;  // A-tasks per plane
  fs.NXT = 3 * (2 * p.nx / FusedShape<LY>::W);  // B-tasks per plane
  fused_lag(grid, fs.NYT + fs.NXT, std::min(fs.NP, p.nz * p.n_items), &fs.D, &fs.S);  // ring <= X1
  fs.slot_elems = 3LL * p.ny * 2 * p.nx;
  if ((e = cudaMemsetAsync(fs.cnt, 0, (1 + 2 * fs.S) * sizeof(int), s))) return e;
  const long long total = (long long)fs.NP * (fs.NYT + fs.NXT);
  k_xyfwd<LX, LY><<<(int)std::min<long long>(grid, total), NT, smem, s>>>(p, fs);
  return cudaGetLastError();
}
static cudaError_t go_xyfwd(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  if (!c->fused_ab || p.x2w != 2 * p.nx || p.k0x != 0) return cudaErrorNotSupported;
  const int LY = 2 * p.ny, LX = 2 * p.nx;
#define IE_FUSED_CASE(a, b) \
  if (LX == a && LY == b) return go_xyfwd_l<a, b>(c, p, s);
  IE_FUSED_CASE(512, 512)
  IE_FUSED_CASE(512, 256)
  IE_FUSED_CASE(256, 256)
  IE_FUSED_CASE(256, 128)
  IE_FUSED_CASE(128, 128)
  IE_FUSED_CASE(128, 64)
  IE_FUSED_CASE(64, 128)
  IE_FUSED_CASE(64, 64)
#undef IE_FUSED_CASE
  return cudaErrorNotSupported;
}

template <int L> static void wrap_xfwd(cudaError_t* e, const ApplyParams& p, cudaStream_t s, int m) { *e = go_xfwd<L>(p, s, m); }
template <int L> static void wrap_yfwd(cudaError_t* e, const ApplyParams& p, cudaStream_t s, int m) { *e = go_yfwd<L>(p, s, m); }
template <int L> static void wrap_zconv(cudaError_t* e, const ApplyParams& p, cudaStream_t s) { *e = go_zconv<L>(p, s); }
template <int L> static void wrap_yinv(cudaError_t* e, const ApplyParams& p, cudaStream_t s) { *e = go_yinv<L>(p, s); }
template <int L> static void wrap_xinv(cudaError_t* e, const ApplyParams& p, cudaStream_t s) { *e = go_xinv<L>(p, s); }

// Profiling: each kernel pass is bracketed by two events on the stream it runs on; a mark
// (kernel id, start event, end event) per bracket.
struct Prof {
  ie_ctx* c;
  cudaError_t take(int n, int* first) {
    if (!c->profiling) return cudaSuccess;
    while (c->ev_pool.size() < c->ev_used + n) {
      cudaEvent_t x;
      cudaError_t e = cudaEventCreate(&x);
      if (e) return e;
      c->ev_pool.push_back(x);
    }
    *first = (int)c->ev_used;
    c->ev_used += n;
    return cudaSuccess;
  }
  void rec(int idx, cudaStream_t s) {
    if (c->profiling) cudaEventRecord(c->ev_pool[idx], s);
  }
  void mark(int kernel, int i0, int i1) {
    if (c->profiling) c->ev_marks.push_back({kernel, i0, i1});
  }
};

static void source_extent(const ApplyParams& p, int* max_rows, int* max_planes) {
  *max_rows = 0;
  *max_planes = 0;
  for (int i = 0; i < p.n_items; ++i) {
    const ApplyItem& it = p.items[i];
    const int rows = (it.sy1 - it.sy0) * (it.sz1 - it.sz0);
    if (rows > *max_rows) *max_rows = rows;
    if (it.sz1 - it.sz0 > *max_planes) *max_planes = it.sz1 - it.sz0;
  }
}

// The five passes in one stream, X2 holding the whole padded grid.
static cudaError_t run_apply(ie_ctx* c, const ApplyParams& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  int max_rows, max_planes;
  source_extent(p, &max_rows, &max_planes);
  Prof pr{c};
  int ev = 0;
  if ((e = pr.take(6, &ev))) return e;
  // items of one launch share the source y/z range (K-A rows, K-B planes)
  pr.rec(ev + 0, s);
  bool ab = false;
  e = go_xyfwd(c, p, s);  // K-AB fused (X1 through an L2-resident ring) where instantiated
  if (e == cudaSuccess) {
    ab = true;
    pr.rec(ev + 2, s);
  } else {
    if (e != cudaErrorNotSupported) return e;
    (void)cudaGetLastError();
    e = cudaSuccess;
    IE_DISPATCH_L(2 * p.nx, wrap_xfwd, &e, p, s, max_rows);
    if (e) return e;
    pr.rec(ev + 1, s);
    IE_DISPATCH_L(2 * p.ny, wrap_yfwd, &e, p, s, max_planes);
    if (e) return e;
    pr.rec(ev + 2, s);
  }
  if (p.mhat) {  // layered background: z-z' contraction per horizontal wavenumber (layered.cu)
    e = launch_zlayer(p, s);
  } else if (const int W16 = zconv16_width(2 * p.nz, 2 * p.nx)) {
    e = go_zconv16(p, s, W16);
  } else {
    IE_DISPATCH_L(2 * p.nz, wrap_zconv, &e, p, s);
  }
  if (e) return e;
  pr.rec(ev + 3, s);
  // forward marks: K-A, K-B separately or K-AB fused; K-C
  auto mark_front = [&]() {
    if (ab) {
      pr.mark(kProfFusedAB, ev + 0, ev + 2);
    } else {
      pr.mark(0, ev + 0, ev + 1);
      pr.mark(1, ev + 1, ev + 2);
    }
    pr.mark(2, ev + 2, ev + 3);
  };
  const int nfront = ab ? 2 : 3;
  e = go_yxinv(c, p, s);  // K-DE fused (X1 through an L2-resident ring) where instantiated
  if (e == cudaSuccess) {
    pr.rec(ev + 4, s);
    mark_front();
    pr.mark(kProfFusedDE, ev + 3, ev + 4);
    c->launches += nfront + 1;
    return e;
  }
  if (e != cudaErrorNotSupported) return e;
  (void)cudaGetLastError();
  e = cudaSuccess;
  IE_DISPATCH_L(2 * p.ny, wrap_yinv, &e, p, s);
  if (e) return e;
  pr.rec(ev + 4, s);
  IE_DISPATCH_L(2 * p.nx, wrap_xinv, &e, p, s);
  pr.rec(ev + 5, s);
  mark_front();
  pr.mark(3, ev + 3, ev + 4);
  pr.mark(4, ev + 4, ev + 5);
  c->launches += nfront + 2;
  return e;
}

// ---------------------------------------------------------------- L2-resident slab pipeline
// For grids whose padded intermediate X2 (192 N bytes per item) is far larger than L2, the
// y-forward, z-convolution and y-inverse passes run slab by slab over S consecutive kx
// columns, each slab's X2 ([item][3][nz][2ny][S]) in a ring of NR buffers small enough to stay
// in the 126 MB L2: K-B(s) writes it, K-C(s) transforms it in place, K-D(s) reads it, and the
// HBM never sees X2 (traffic per apply 576 N + |G| instead of 1344 N + |G| bytes).  The three
// passes run on three streams ordered by events, so slab s+1's K-B overlaps slab s's K-C and
// slab s-1's K-D.
constexpr int kSlabRing = 3;
constexpr size_t kSlabL2Budget = 80ull << 20;  // bytes of X2 ring kept in flight

static int slab_width(const ApplyParams& p) {
  if (p.mhat) return 0;
  const int Lx = 2 * p.nx;
  const int W16 = zconv16_width(2 * p.nz, Lx);
  if (!W16) return 0;
  const int Ty = (2 * p.ny) / std::min(8, 2 * p.ny);  // threads per y-line (FftPlan<2ny>::T)
  const int Wy = y_width(Ty, Lx);                     // K-B / K-D tile width
  const int S = std::max(W16, Wy);
  if (S > Lx || Lx % S) return 0;
  const size_t full = (size_t)p.n_items * 3 * p.nz * 2 * p.ny * Lx * sizeof(double2);
  const size_t slab = (size_t)p.n_items * 3 * p.nz * 2 * p.ny * S * sizeof(double2);
  if (full <= 2 * kSlabL2Budget || kSlabRing * slab > kSlabL2Budget) return 0;
  return S;
}

static cudaError_t ensure_aux(ie_ctx* c) {
  if (c->aux_ready) return cudaSuccess;
  cudaError_t e;
  for (int i = 0; i < 3; ++i)
    if ((e = cudaStreamCreateWithFlags(&c->aux[i], cudaStreamNonBlocking))) return e;
  for (int i = 0; i < 1 + 3 * kSlabRing; ++i)
    if ((e = cudaEventCreateWithFlags(&c->aux_ev[i], cudaEventDisableTiming))) return e;
  c->aux_ready = true;
  return cudaSuccess;
}

static cudaError_t run_apply_slabs(ie_ctx* c, const ApplyParams& p, cudaStream_t s, int S) {
  cudaError_t e = cudaSuccess;
  if ((e = ensure_aux(c))) return e;
  int max_rows, max_planes;
  source_extent(p, &max_rows, &max_planes);
  const int Lx = 2 * p.nx, nslab = Lx / S;
  const long long slab_elems = (long long)p.n_items * 3 * p.nz * 2 * p.ny * S;
  cudaEvent_t evA = c->aux_ev[0];
  cudaEvent_t* evB = c->aux_ev + 1;
  cudaEvent_t* evC = c->aux_ev + 1 + kSlabRing;
  cudaEvent_t* evD = c->aux_ev + 1 + 2 * kSlabRing;
  cudaStream_t sB = c->aux[0], sC = c->aux[1], sD = c->aux[2];
  Prof pr{c};
  int ev = 0;
  if ((e = pr.take(4 + 6 * nslab, &ev))) return e;
  pr.rec(ev + 0, s);
  IE_DISPATCH_L(2 * p.nx, wrap_xfwd, &e, p, s, max_rows);
  if (e) return e;
  pr.rec(ev + 1, s);
  pr.mark(0, ev + 0, ev + 1);
  if ((e = cudaEventRecord(evA, s))) return e;
  for (cudaStream_t x : {sB, sC, sD})
    if ((e = cudaStreamWaitEvent(x, evA, 0))) return e;
  for (int sl = 0; sl < nslab; ++sl) {
    const int b = sl % kSlabRing;
    ApplyParams q = p;
    q.X2 = p.X2 + b * slab_elems;
    q.x2w = S;
    q.k0x = sl * S;
    const int e0 = ev + 4 + 6 * sl;
    if (sl >= kSlabRing && (e = cudaStreamWaitEvent(sB, evD[b], 0))) return e;  // buffer b free
    pr.rec(e0 + 0, sB);
    IE_DISPATCH_L(2 * p.ny, wrap_yfwd, &e, q, sB, max_planes);
    if (e) return e;
    pr.rec(e0 + 1, sB);
    if ((e = cudaEventRecord(evB[b], sB)) || (e = cudaStreamWaitEvent(sC, evB[b], 0))) return e;
    pr.rec(e0 + 2, sC);
    if ((e = go_zconv16(q, sC, zconv16_width(2 * p.nz, Lx)))) return e;
    pr.rec(e0 + 3, sC);
    if ((e = cudaEventRecord(evC[b], sC)) || (e = cudaStreamWaitEvent(sD, evC[b], 0))) return e;
    pr.rec(e0 + 4, sD);
    IE_DISPATCH_L(2 * p.ny, wrap_yinv, &e, q, sD);
    if (e) return e;
    pr.rec(e0 + 5, sD);
    if ((e = cudaEventRecord(evD[b], sD))) return e;
    pr.mark(1, e0 + 0, e0 + 1);
    pr.mark(2, e0 + 2, e0 + 3);
    pr.mark(3, e0 + 4, e0 + 5);
  }
  if ((e = cudaStreamWaitEvent(s, evD[(nslab - 1) % kSlabRing], 0))) return e;
  pr.rec(ev + 2, s);
  IE_DISPATCH_L(2 * p.nx, wrap_xinv, &e, p, s);
  pr.rec(ev + 3, s);
  pr.mark(4, ev + 2, ev + 3);
  c->launches += 2 + 3 * nslab;
  return e;
}

ie_status launch_apply(ie_ctx* c, ApplyParams& p) {
  if (p.n_items <= 0) return IE_OK;
  if (p.n_items > kMaxItems) return fail(c, IE_ERR_INVALID_ARGUMENT, "internal: too many apply items");
  for (int i = 1; i < p.n_items; ++i)
    if (p.items[i].sz0 != p.items[0].sz0 || p.items[i].sz1 != p.items[0].sz1 ||
        p.items[i].sy0 != p.items[0].sy0 || p.items[i].sy1 != p.items[0].sy1)
      return fail(c, IE_ERR_INVALID_ARGUMENT, "internal: batched apply items must share the source y/z range");
  p.tw_x = c->tw.get(2 * p.nx, 0);
  p.tw_y = c->tw.get(2 * p.ny, 0);
  p.tw_z = c->tw.get(2 * p.nz, 0);
  p.tw_zr = c->tw.get(2 * p.nz, 1);
  p.pw_z = c->tw.powers(2 * p.nz);
  p.x2w = 2 * p.nx;
  p.k0x = 0;
  const int S = c->slabs ? slab_width(p) : 0;  // off unless IE_SLABS=1 (measured slower)
  cudaError_t e = S ? run_apply_slabs(c, p, c->stream, S) : run_apply(c, p, c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "operator kernels");
  return IE_OK;
}

}  // namespace ie
