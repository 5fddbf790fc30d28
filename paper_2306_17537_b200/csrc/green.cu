// A0: the discrete Green kernel and its packed 2x-padded spectrum (Eq. 5, 7, 10).
//
// For a domain of (nx,ny,nz) cells the kernel K(d) = G^E(d h) dv (midpoint rule) for
// d != 0 and the equivolume-sphere self term for d = 0 (reading R3) is sampled on
// the circulant embedding of size (2nx,2ny,2nz) -- index i holds offset i (i < n), 0 at
// i = n, i - 2n (i > n) -- for each of the six unique components (xx,yy,zz,xy,xz,yz),
// transformed by a full 3-D FFT (generic in-place line FFTs below), and packed to the
// octant [0,n]^3 (the spectrum is even/odd per axis) with the 1/(8 nx ny nz) inverse-FFT
// normalisation folded in.  One-off per (grid shape, sigma0, f); not on the hot loop.
#include <math.h>

#include <algorithm>

#include "fft_core.cuh"
#include "ie_internal.h"
#include "kernel_eval.cuh"

namespace ie {

// K_comp at circulant index (ix,iy,iz) of the (2nx,2ny,2nz) grid, comp in 0..5
__global__ void k_green_sample(double2* __restrict__ C, GreenArgs a, int comp) {
  const long long Lx = 2 * a.nx, Ly = 2 * a.ny, Lz = 2 * a.nz;
  const long long total = Lx * Ly * Lz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(e % Lx), iy = (int)((e / Lx) % Ly), iz = (int)(e / (Lx * Ly));
    double2 out = make_double2(0.0, 0.0);
    if (ix != a.nx && iy != a.ny && iz != a.nz) {
      const int dxi = ix < a.nx ? ix : ix - (int)Lx;
      const int dyi = iy < a.ny ? iy : iy - (int)Ly;
      const int dzi = iz < a.nz ? iz : iz - (int)Lz;
      out = kernel_sample(a, dxi, dyi, dzi, comp);
    }
    C[e] = out;
  }
}

// Generic in-place forward FFT of length L along the middle axis of a [outer][L][inner]
// array (no zero-padding, no pruning).  CTA = LPC lines x W columns.
template <int L>
__global__ void __launch_bounds__(512) k_fft_axis(double2* __restrict__ data, long long inner, long long outer,
                                                  const double2* __restrict__ tw, int W) {
  using P = FftPlan<L>;
  constexpr int T = P::T, V = P::V, R0 = P::radix(0, false), RL = P::radix(P::NST - 1, false);
  extern __shared__ double2 sm[];
  const int lpc = blockDim.x / (T * W);
  const int c = threadIdx.x % W, t = (threadIdx.x / W) % T, lo = threadIdx.x / (W * T);
  const long long ncb = (inner + W - 1) / W;  // column blocks; flattened grid (x dim holds 2^31)
  const long long line = (long long)(blockIdx.x / ncb) * lpc + lo;
  const long long col = (long long)(blockIdx.x % ncb) * W + c;
  const bool valid = line < outer && col < inner;
  double2* base = data + line * L * inner + col;
  double2 v[1][V];
#pragma unroll
  for (int u = 0; u < V / R0; ++u)
#pragma unroll
    for (int r = 0; r < R0; ++r)
      v[0][u * R0 + r] = valid ? base[(long long)(t + u * T + r * (L / R0)) * inner] : czero();
  const int region = padded(L * W);
  auto idx = [&](int) { return SIdx{lo * region, W, c}; };
  fft_run<L, false, -1, 1>(v, sm, idx, t, tw, false);
  if (!valid) return;
#pragma unroll
  for (int u = 0; u < V / RL; ++u)
#pragma unroll
    for (int r = 0; r < RL; ++r) base[(long long)(t + u * T + r * (L / RL)) * inner] = v[0][u * RL + r];
}

__global__ void k_green_pack(const double2* __restrict__ C, double2* __restrict__ oct, int nx, int ny, int nz,
                             double scale) {
  const long long Ox = nx + 1, Oy = ny + 1, Oz = nz + 1, total = Ox * Oy * Oz;
  const long long Lx = 2 * nx, Ly = 2 * ny;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long ix = e % Ox, iy = (e / Ox) % Oy, iz = e / (Ox * Oy);
    const double2 v = C[(iz * Ly + iy) * Lx + ix];
    oct[e] = make_double2(v.x * scale, v.y * scale);
  }
}

template <int L>
static cudaError_t fft_axis_launch(double2* data, long long inner, long long outer, const double2* tw,
                                   cudaStream_t s) {
  constexpr int T = FftPlan<L>::T;
  const int wmax = 512 / T;
  const int W = (inner >= 8) ? (int)std::min<long long>(inner, std::max(std::min(8, wmax), 256 / T)) : 1;
  int lpc = (inner >= 8) ? 1 : std::max(1, 128 / T);
  if (W * T > 512) return cudaErrorInvalidConfiguration;
  const size_t smem = (size_t)lpc * padded(L * W) * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_fft_axis<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e) return e;
  }
  dim3 grid((unsigned)(((inner + W - 1) / W) * ((outer + lpc - 1) / lpc)));
  k_fft_axis<L><<<grid, lpc * T * W, smem, s>>>(data, inner, outer, tw, W);
  return cudaGetLastError();
}

cudaError_t fft_axis(int L, double2* data, long long inner, long long outer, const double2* tw,
                            cudaStream_t s) {
  switch (L) {
    case 2: return fft_axis_launch<2>(data, inner, outer, tw, s);
    case 4: return fft_axis_launch<4>(data, inner, outer, tw, s);
    case 8: return fft_axis_launch<8>(data, inner, outer, tw, s);
    case 16: return fft_axis_launch<16>(data, inner, outer, tw, s);
    case 32: return fft_axis_launch<32>(data, inner, outer, tw, s);
    case 64: return fft_axis_launch<64>(data, inner, outer, tw, s);
    case 128: return fft_axis_launch<128>(data, inner, outer, tw, s);
    case 256: return fft_axis_launch<256>(data, inner, outer, tw, s);
    case 512: return fft_axis_launch<512>(data, inner, outer, tw, s);
    case 1024: return fft_axis_launch<1024>(data, inner, outer, tw, s);
  }
  return cudaErrorInvalidValue;
}

GreenArgs green_args(const ie_ctx* c, int nx, int ny, int nz) {
  GreenArgs a;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.dx = c->g.dx;
  a.dy = c->g.dy;
  a.dz = c->g.dz;
  a.dv = c->g.dx * c->g.dy * c->g.dz;
  a.k0r = c->k0.real();
  a.k0i = c->k0.imag();
  a.sigma_b = c->sigma_b;
  a.selfr = c->self.real();
  a.selfi = c->self.imag();
  return a;
}

ie_status build_green(ie_ctx* c, int nx, int ny, int nz, GreenSpec* out) {
  const GreenArgs a = green_args(c, nx, ny, nz);
  const long long Lx = 2 * nx, Ly = 2 * ny, Lz = 2 * nz, total = Lx * Ly * Lz;
  const long long ooct = (long long)(nx + 1) * (ny + 1) * (nz + 1);
  out->nx = nx;
  out->ny = ny;
  out->nz = nz;
  IE_CUDA(c, cudaMalloc(&out->oct, 6 * ooct * sizeof(double2)));
  double2* C = nullptr;
  IE_CUDA(c, cudaMalloc(&C, total * sizeof(double2)));
  const double scale = 1.0 / (double)total;
  cudaError_t e = cudaSuccess;
  for (int comp = 0; comp < 6 && e == cudaSuccess; ++comp) {
    k_green_sample<<<1184, 256, 0, c->stream>>>(C, a, comp);
    c->launches++;
    e = cudaGetLastError();
    if (!e) e = fft_axis((int)Lx, C, 1, Ly * Lz, c->tw.get((int)Lx, 0), c->stream);
    if (!e) e = fft_axis((int)Ly, C, Lx, Lz, c->tw.get((int)Ly, 0), c->stream);
    if (!e) e = fft_axis((int)Lz, C, Lx * Ly, 1, c->tw.get((int)Lz, 0), c->stream);
    c->launches += 3;
    if (!e) {
      k_green_pack<<<1184, 256, 0, c->stream>>>(C, out->oct + comp * ooct, nx, ny, nz, scale);
      c->launches++;
      e = cudaGetLastError();
    }
  }
  if (!e) e = cudaStreamSynchronize(c->stream);
  cudaFree(C);
  if (e) return cuda_fail(c, e, "green spectrum setup");
  return IE_OK;
}

const GreenSpec* green_for(ie_ctx* c, int nx, int ny, int nz, int k0, ie_status* st) {
  *st = IE_OK;
  if (!c->layered) k0 = 0;  // homogeneous spectra depend on the shape only
  for (auto& g : c->greens)
    if (g.nx == nx && g.ny == ny && g.nz == nz && g.k0 == k0) return &g;
  GreenSpec gs;
  *st = c->layered ? build_layer_spec(c, nx, ny, nz, k0, &gs) : build_green(c, nx, ny, nz, &gs);
  if (*st != IE_OK) return nullptr;
  c->greens.push_back(gs);
  return &c->greens.back();
}

}  // namespace ie
