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

namespace ie {

struct GreenArgs {
  int nx, ny, nz;
  double dx, dy, dz, dv;
  double k0r, k0i, sigma_b;
  double selfr, selfi;
};

// complex helpers on (re, im) doubles
__device__ __forceinline__ double2 cexp_i(double2 z) {  // exp(i z)
  const double m = exp(-z.y);
  double s, c;
  sincos(z.x, &s, &c);
  return make_double2(m * c, m * s);
}

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
      if (dxi == 0 && dyi == 0 && dzi == 0) {
        if (comp < 3) out = make_double2(a.selfr, a.selfi);
      } else {
        const double X = dxi * a.dx, Y = dyi * a.dy, Z = dzi * a.dz;
        const double R = sqrt(X * X + Y * Y + Z * Z);
        const double iR = 1.0 / R;
        // g = exp(i k0 R) / (4 pi R)
        const double2 e1 = cexp_i(make_double2(a.k0r * R, a.k0i * R));
        const double2 g = make_double2(e1.x * iR / (4.0 * kPi), e1.y * iR / (4.0 * kPi));
        // k0^2, i k0 / R
        const double2 k2 = make_double2(a.k0r * a.k0r - a.k0i * a.k0i, 2.0 * a.k0r * a.k0i);
        const double2 ikR = make_double2(-a.k0i * iR, a.k0r * iR);
        // alpha = k0^2 + i k0/R - 1/R^2 ; beta = 3/R^2 - 3 i k0/R - k0^2
        const double2 al = make_double2(k2.x + ikR.x - iR * iR, k2.y + ikR.y);
        const double2 be = make_double2(3.0 * iR * iR - 3.0 * ikR.x - k2.x, -3.0 * ikR.y - k2.y);
        double hp, hq;
        const double hx = X * iR, hy = Y * iR, hz = Z * iR;
        bool diag = comp < 3;
        switch (comp) {
          case 0: hp = hx; hq = hx; break;
          case 1: hp = hy; hq = hy; break;
          case 2: hp = hz; hq = hz; break;
          case 3: hp = hx; hq = hy; break;
          case 4: hp = hx; hq = hz; break;
          default: hp = hy; hq = hz; break;
        }
        double2 coef = make_double2(be.x * hp * hq, be.y * hp * hq);
        if (diag) coef = make_double2(coef.x + al.x, coef.y + al.y);
        const double s = a.dv / a.sigma_b;
        out = make_double2((coef.x * g.x - coef.y * g.y) * s, (coef.x * g.y + coef.y * g.x) * s);
      }
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

static cudaError_t fft_axis(int L, double2* data, long long inner, long long outer, const double2* tw,
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

ie_status build_green(ie_ctx* c, int nx, int ny, int nz, GreenSpec* out) {
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

const GreenSpec* green_for(ie_ctx* c, int nx, int ny, int nz, ie_status* st) {
  *st = IE_OK;
  for (auto& g : c->greens)
    if (g.nx == nx && g.ny == ny && g.nz == nz) return &g;
  GreenSpec gs;
  *st = build_green(c, nx, ny, nz, &gs);
  if (*st != IE_OK) return nullptr;
  c->greens.push_back(gs);
  return &c->greens.back();
}

}  // namespace ie
