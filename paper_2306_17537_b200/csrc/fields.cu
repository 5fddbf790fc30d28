// Per-cell field kernels: contrast packing, incident field E0 of magnetic dipoles
// (Eq. 3's E^(0), reading R4), receiver magnetic fields (Eq. 4 with Eq. 6), box
// gather/scatter for the DD blocks (Eq. 16), axpby and deterministic norms (Eq. 9).
#include <math.h>

#include <algorithm>
#include <vector>

#include "fft_core.cuh"
#include "ie_internal.h"

namespace ie {

static inline unsigned grid_for(long long n, int block, int cap = 148 * 16) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ------------------------------------------------------------------- contrast
// FULL9 cell-major [N][3][3] -> dsigma SYM6 SoA [6][N] = sigma - sigma_b I; flags asymmetry.
// sbz (layered backgrounds): sigma_b of each cell layer, indexed c / nxy; else sb for all
__global__ void k_contrast_full9(const double* __restrict__ s, double* __restrict__ ds, long long N, double sb0,
                                 const double* __restrict__ sbz, long long nxy, int* __restrict__ bad) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
    const double sb = sbz ? sbz[c / nxy] : sb0;
    const double* m = s + 9 * c;
    const double xx = m[0], xy = m[1], xz = m[2], yx = m[3], yy = m[4], yz = m[5], zx = m[6], zy = m[7], zz = m[8];
    const double mx = fmax(fmax(fabs(xx), fabs(yy)), fmax(fabs(zz), fmax(fabs(xy), fmax(fabs(xz), fabs(yz)))));
    const double tol = 1e-12 * mx;
    if (fabs(xy - yx) > tol || fabs(xz - zx) > tol || fabs(yz - zy) > tol || !isfinite(mx)) atomicOr(bad, 1);
    ds[c] = xx - sb;
    ds[N + c] = yy - sb;
    ds[2 * N + c] = zz - sb;
    ds[3 * N + c] = xy;
    ds[4 * N + c] = xz;
    ds[5 * N + c] = yz;
  }
}
__global__ void k_contrast_sym6(const double* __restrict__ s, double* __restrict__ ds, long long N, double sb0,
                                const double* __restrict__ sbz, long long nxy, int* __restrict__ bad) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
    const double sb = sbz ? sbz[c / nxy] : sb0;
    for (int k = 0; k < 6; ++k) {
      const double v = s[k * N + c];
      if (!isfinite(v)) atomicOr(bad, 1);
      ds[k * N + c] = v - (k < 3 ? sb : 0.0);
    }
  }
}

ie_status pack_contrast(ie_ctx* c, const void* sigma_dev, int layout) {
  const long long N = (long long)c->g.nx * c->g.ny * c->g.nz;
  // pack into a fresh buffer: a rejected conductivity leaves the context's contrast untouched
  double* dnew = nullptr;
  IE_CUDA(c, cudaMalloc(&dnew, 6 * N * sizeof(double)));
  int* bad = nullptr;
  double* sbz = nullptr;  // per-layer background (P:48 with sigma_b(z); reading R17)
  IE_CUDA(c, cudaMalloc(&bad, 8 + (c->layered ? c->g.nz * sizeof(double) : 0)));
  IE_CUDA(c, cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  std::vector<double> hsb;
  if (c->layered) {
    for (int k = 0; k < c->g.nz; ++k) hsb.push_back(sigma_b_at(c, k));
    sbz = (double*)((char*)bad + 8);
    IE_CUDA(c, cudaMemcpyAsync(sbz, hsb.data(), hsb.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  const long long nxy = (long long)c->g.nx * c->g.ny;
  if (layout == 0)
    k_contrast_full9<<<grid_for(N, 256), 256, 0, c->stream>>>((const double*)sigma_dev, dnew, N, c->sigma_b, sbz,
                                                              nxy, bad);
  else
    k_contrast_sym6<<<grid_for(N, 256), 256, 0, c->stream>>>((const double*)sigma_dev, dnew, N, c->sigma_b, sbz,
                                                             nxy, bad);
  c->launches++;
  int hbad = 0;
  cudaError_t e = cudaGetLastError();
  if (!e) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  cudaFree(bad);
  if (e || hbad) cudaFree(dnew);
  if (e) return cuda_fail(c, e, "set_contrast");
  if (hbad) return fail(c, IE_ERR_INVALID_ARGUMENT, "sigma is not symmetric to 1e-12 (P:415) or not finite");
  cudaFree(c->dsig);
  c->dsig = dnew;
  c->contrast_set = true;
  if (c->pre_p) {  // a new contrast invalidates the preconditioner (rebuilt on next use)
    cudaFree(c->pre_p);
    c->pre_p = c->pre_a = c->pre_dp = nullptr;
  }
  return IE_OK;
}

// ------------------------------------------------------------ incident field (E^(0))
struct IncArgs {
  int nx, ny, nz;
  double ox, oy, oz, dx, dy, dz;
  double k0r, k0i, omega_mu0;
  double sx, sy, sz, mx, my, mz;
};
// E0 = i omega mu0 g (i k0 - 1/R) (Rhat x m),  R = r - r_s
__global__ void k_incident(double2* __restrict__ E, IncArgs a) {
  const long long N = (long long)a.nx * a.ny * a.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(c % a.nx), iy = (int)((c / a.nx) % a.ny), iz = (int)(c / ((long long)a.nx * a.ny));
    const double X = a.ox + ix * a.dx - a.sx, Y = a.oy + iy * a.dy - a.sy, Z = a.oz + iz * a.dz - a.sz;
    const double R = sqrt(X * X + Y * Y + Z * Z), iR = 1.0 / R;
    const double m = exp(-a.k0i * R);
    double sn, cs;
    sincos(a.k0r * R, &sn, &cs);
    const double2 g = make_double2(m * cs * iR / (4 * kPi), m * sn * iR / (4 * kPi));
    const double2 f = make_double2(-a.k0i - iR, a.k0r);            // i k0 - 1/R
    const double2 gf = cmul(g, f);
    const double2 coef = make_double2(-a.omega_mu0 * gf.y, a.omega_mu0 * gf.x);  // i omega mu0 * gf
    const double hx = X * iR, hy = Y * iR, hz = Z * iR;
    const double cx = hy * a.mz - hz * a.my, cy = hz * a.mx - hx * a.mz, cz = hx * a.my - hy * a.mx;
    E[c] = cscale(coef, cx);
    E[N + c] = cscale(coef, cy);
    E[2 * N + c] = cscale(coef, cz);
  }
}

ie_status compute_incident(ie_ctx* c, int n_src, const double* pos, const double* moment, double2* out) {
  const long long N = (long long)c->g.nx * c->g.ny * c->g.nz;
  const double hmin = std::min(c->g.dx, std::min(c->g.dy, c->g.dz));
  for (int s = 0; s < n_src; ++s) {
    // placement: nearest centroid distance (E0 singular at R = 0)
    double d2 = 0;
    const double h[3] = {c->g.dx, c->g.dy, c->g.dz};
    const int n[3] = {c->g.nx, c->g.ny, c->g.nz};
    for (int a = 0; a < 3; ++a) {
      double t = (pos[3 * s + a] - c->g.origin[a]) / h[a];
      double k = std::min(std::max(std::round(t), 0.0), (double)(n[a] - 1));
      const double dd = (t - k) * h[a];
      d2 += dd * dd;
    }
    if (sqrt(d2) < 1e-6 * hmin) return fail(c, IE_ERR_PLACEMENT, "source within 1e-6*h of a cell centroid");
    IncArgs a;
    a.nx = c->g.nx;
    a.ny = c->g.ny;
    a.nz = c->g.nz;
    a.ox = c->g.origin[0];
    a.oy = c->g.origin[1];
    a.oz = c->g.origin[2];
    a.dx = c->g.dx;
    a.dy = c->g.dy;
    a.dz = c->g.dz;
    a.k0r = c->k0.real();
    a.k0i = c->k0.imag();
    a.omega_mu0 = c->omega * kMu0;
    a.sx = pos[3 * s];
    a.sy = pos[3 * s + 1];
    a.sz = pos[3 * s + 2];
    a.mx = moment[3 * s];
    a.my = moment[3 * s + 1];
    a.mz = moment[3 * s + 2];
    k_incident<<<grid_for(N, 256), 256, 0, c->stream>>>(out + (long long)s * 3 * N, a);
    IE_CHECK_LAUNCH(c, "k_incident");
  }
  return IE_OK;
}

// ------------------------------------------------------------------ receivers (Eq. 4)
struct RxArgs {
  int nx, ny, nz;
  double ox, oy, oz, dx, dy, dz, dv;
  double k0r, k0i;
  double rx, ry, rz;
  long long N;
};
// partial sums over a chunk of cells of grad g(r - r_c) x (dsigma_c E_c) dv
__global__ void __launch_bounds__(256) k_rx_partial(const double2* __restrict__ E, const double* __restrict__ ds,
                                                    RxArgs a, double2* __restrict__ part) {
  const long long N = a.N;
  double2 acc[3] = {czero(), czero(), czero()};
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(c % a.nx), iy = (int)((c / a.nx) % a.ny), iz = (int)(c / ((long long)a.nx * a.ny));
    const double X = a.rx - (a.ox + ix * a.dx), Y = a.ry - (a.oy + iy * a.dy), Z = a.rz - (a.oz + iz * a.dz);
    const double R2 = X * X + Y * Y + Z * Z;
    if (R2 == 0.0) continue;  // odd kernel over the equivolume ball: no self term
    const double sxx = ds[c], syy = ds[N + c], szz = ds[2 * N + c], sxy = ds[3 * N + c], sxz = ds[4 * N + c],
                 syz = ds[5 * N + c];
    if (sxx == 0.0 && syy == 0.0 && szz == 0.0 && sxy == 0.0 && sxz == 0.0 && syz == 0.0) continue;
    const double2 e0 = E[c], e1 = E[N + c], e2 = E[2 * N + c];
    const double2 J0 = make_double2(sxx * e0.x + sxy * e1.x + sxz * e2.x, sxx * e0.y + sxy * e1.y + sxz * e2.y);
    const double2 J1 = make_double2(sxy * e0.x + syy * e1.x + syz * e2.x, sxy * e0.y + syy * e1.y + syz * e2.y);
    const double2 J2 = make_double2(sxz * e0.x + syz * e1.x + szz * e2.x, sxz * e0.y + syz * e1.y + szz * e2.y);
    const double R = sqrt(R2), iR = 1.0 / R;
    const double m = exp(-a.k0i * R);
    double sn, cs;
    sincos(a.k0r * R, &sn, &cs);
    const double2 g = make_double2(m * cs * iR / (4 * kPi), m * sn * iR / (4 * kPi));
    const double2 f = make_double2(-a.k0i - iR, a.k0r);
    const double2 gf = cscale(cmul(g, f), a.dv);
    const double hx = X * iR, hy = Y * iR, hz = Z * iR;
    // (Rhat x J)
    const double2 c0 = make_double2(hy * J2.x - hz * J1.x, hy * J2.y - hz * J1.y);
    const double2 c1 = make_double2(hz * J0.x - hx * J2.x, hz * J0.y - hx * J2.y);
    const double2 c2 = make_double2(hx * J1.x - hy * J0.x, hx * J1.y - hy * J0.y);
    acc[0] = cadd(acc[0], cmul(gf, c0));
    acc[1] = cadd(acc[1], cmul(gf, c1));
    acc[2] = cadd(acc[2], cmul(gf, c2));
  }
  __shared__ double2 red[3][256];
  for (int k = 0; k < 3; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] = cadd(red[k][threadIdx.x], red[k][threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) part[blockIdx.x * 3 + k] = red[k][0];
}

// H0 = (k0^2 + grad grad) g m at r, added to the reduced partials (one thread)
struct H0Args {
  double k0r, k0i, X, Y, Z, mx, my, mz;
};
__global__ void k_rx_finish(const double2* __restrict__ part, int nblk, H0Args h, double2* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double2 s[3] = {czero(), czero(), czero()};
  for (int b = 0; b < nblk; ++b)
    for (int k = 0; k < 3; ++k) s[k] = cadd(s[k], part[b * 3 + k]);
  const double R = sqrt(h.X * h.X + h.Y * h.Y + h.Z * h.Z), iR = 1.0 / R;
  const double m = exp(-h.k0i * R);
  double sn, cs;
  sincos(h.k0r * R, &sn, &cs);
  const double2 g = make_double2(m * cs * iR / (4 * kPi), m * sn * iR / (4 * kPi));
  const double2 k2 = make_double2(h.k0r * h.k0r - h.k0i * h.k0i, 2 * h.k0r * h.k0i);
  const double2 ikR = make_double2(-h.k0i * iR, h.k0r * iR);
  const double2 al = cmul(make_double2(k2.x + ikR.x - iR * iR, k2.y + ikR.y), g);
  const double2 be = cmul(make_double2(3 * iR * iR - 3 * ikR.x - k2.x, -3 * ikR.y - k2.y), g);
  const double hx = h.X * iR, hy = h.Y * iR, hz = h.Z * iR;
  const double rm = hx * h.mx + hy * h.my + hz * h.mz;
  const double mm[3] = {h.mx, h.my, h.mz}, hh[3] = {hx, hy, hz};
  for (int k = 0; k < 3; ++k) {
    const double2 h0 = cadd(cscale(al, mm[k]), cscale(be, hh[k] * rm));
    out[k] = cadd(s[k], h0);
  }
}

ie_status receivers(ie_ctx* c, const double2* e, int n_rx, const double* rx, cplx* h_out, const double* src_pos,
                    const double* src_mom, int n_src, double2* scratch) {
  const long long N = (long long)c->g.nx * c->g.ny * c->g.nz;
  const int nblk = 296;
  double2* part = scratch;                       // [nblk][3]
  double2* res = scratch + (size_t)nblk * 3;     // [n_src][n_rx][3]
  for (int s = 0; s < n_src; ++s)
    for (int r = 0; r < n_rx; ++r) {
      RxArgs a;
      a.nx = c->g.nx;
      a.ny = c->g.ny;
      a.nz = c->g.nz;
      a.ox = c->g.origin[0];
      a.oy = c->g.origin[1];
      a.oz = c->g.origin[2];
      a.dx = c->g.dx;
      a.dy = c->g.dy;
      a.dz = c->g.dz;
      a.dv = c->g.dx * c->g.dy * c->g.dz;
      a.k0r = c->k0.real();
      a.k0i = c->k0.imag();
      a.rx = rx[3 * r];
      a.ry = rx[3 * r + 1];
      a.rz = rx[3 * r + 2];
      a.N = N;
      k_rx_partial<<<nblk, 256, 0, c->stream>>>(e + (long long)s * 3 * N, c->dsig, a, part);
      IE_CHECK_LAUNCH(c, "k_rx_partial");
      H0Args h;
      h.k0r = a.k0r;
      h.k0i = a.k0i;
      h.X = a.rx - src_pos[3 * s];
      h.Y = a.ry - src_pos[3 * s + 1];
      h.Z = a.rz - src_pos[3 * s + 2];
      h.mx = src_mom[3 * s];
      h.my = src_mom[3 * s + 1];
      h.mz = src_mom[3 * s + 2];
      k_rx_finish<<<1, 32, 0, c->stream>>>(part, nblk, h, res + ((size_t)s * n_rx + r) * 3);
      IE_CHECK_LAUNCH(c, "k_rx_finish");
    }
  std::vector<double2> host((size_t)n_src * n_rx * 3);
  IE_CUDA(c, cudaMemcpyAsync(host.data(), res, host.size() * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  for (size_t i = 0; i < host.size(); ++i) h_out[i] = cplx(host[i].x, host[i].y);
  return IE_OK;
}

// ---------------------------------------------------------------- gather / scatter
// full: [nsys][3][nz][ny][nx] (stride full_stride per system); box: [nsys][3][bz][by][bx]
__global__ void k_box_copy(double2* __restrict__ full, double2* __restrict__ box, int nx, int ny, int nz, ie_box b,
                           long long fstride, long long bstride, int to_box) {
  const int bx = b.i1 - b.i0, by = b.j1 - b.j0, bz = b.k1 - b.k0;
  const long long Nb = (long long)bx * by * bz, Nf = (long long)nx * ny * nz;
  const long long total = 3 * Nb;
  const int s = blockIdx.y;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / Nb);
    const long long r = e % Nb;
    const int ix = (int)(r % bx), iy = (int)((r / bx) % by), iz = (int)(r / ((long long)bx * by));
    const long long f = q * Nf + ((long long)(iz + b.k0) * ny + (iy + b.j0)) * nx + (ix + b.i0);
    if (to_box) box[s * bstride + e] = full[s * fstride + f];
    else full[s * fstride + f] = box[s * bstride + e];
  }
}

void launch_gather(ie_ctx* c, const double2* full, double2* box, const ie_box& b, int nsys, long long fstride,
                   long long bstride) {
  const long long n = 3LL * (b.i1 - b.i0) * (b.j1 - b.j0) * (b.k1 - b.k0);
  k_box_copy<<<dim3(grid_for(n, 256, 1184), nsys), 256, 0, c->stream>>>((double2*)full, box, c->g.nx, c->g.ny,
                                                                         c->g.nz, b, fstride, bstride, 1);
  c->launches++;
}
void launch_scatter(ie_ctx* c, double2* full, const double2* box, const ie_box& b, int nsys, long long fstride,
                    long long bstride) {
  const long long n = 3LL * (b.i1 - b.i0) * (b.j1 - b.j0) * (b.k1 - b.k0);
  k_box_copy<<<dim3(grid_for(n, 256, 1184), nsys), 256, 0, c->stream>>>(full, (double2*)box, c->g.nx, c->g.ny,
                                                                         c->g.nz, b, fstride, bstride, 0);
  c->launches++;
}

// z = a x + b y (y may be null)
// called in place (z == x or z == y): no __restrict__ on the three vectors (each element is read
// and written by the same thread)
__global__ void k_axpby(double2* z, double2 a, const double2* x, double2 b, const double2* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = cmul(a, x[i]);
    if (y) v = cadd(v, cmul(b, y[i]));
    z[i] = v;
  }
}
void launch_axpby(ie_ctx* c, double2* z, cplx a, const double2* x, cplx b, const double2* y, long long n) {
  k_axpby<<<grid_for(n, 256, 148 * 8), 256, 0, c->stream>>>(z, make_double2(a.real(), a.imag()), x,
                                                           make_double2(b.real(), b.imag()), y, n);
  c->launches++;
}

// ---------------------------------------- contraction-IE right preconditioner
// Per cell, from dsigma (sym6) and sigma_b(z):  a = (sigma + sigma_b I) / (2 sigma_b),
// P = a^-1 = 2 sigma_b (sigma + sigma_b I)^-1 and dsigma P (a function of the same symmetric
// matrix as dsigma, hence symmetric).  The change of unknown chi = a E turns Eq. 8 into
// (I - G dsigma) P chi = E0 with the same Eq. 9 residual (Hursan & Zhdanov's contraction IE as
// a right preconditioner).
__global__ void k_precond_build(const double* __restrict__ ds, double* __restrict__ pa, double* __restrict__ pp,
                                double* __restrict__ pdp, long long N, long long nxy, double sb0,
                                const double* __restrict__ sbz) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
    const double sb = sbz ? sbz[c / nxy] : sb0;
    const double d[6] = {ds[c], ds[N + c], ds[2 * N + c], ds[3 * N + c], ds[4 * N + c], ds[5 * N + c]};
    // a = (dsigma + 2 sigma_b I) / (2 sigma_b)  (sigma + sigma_b I = dsigma + 2 sigma_b I)
    const double s = 0.5 / sb;
    const double a0 = (d[0] + 2 * sb) * s, a1 = (d[1] + 2 * sb) * s, a2 = (d[2] + 2 * sb) * s;
    const double a3 = d[3] * s, a4 = d[4] * s, a5 = d[5] * s;  // xy, xz, yz
    // symmetric inverse by cofactors
    const double c00 = a1 * a2 - a5 * a5, c11 = a0 * a2 - a4 * a4, c22 = a0 * a1 - a3 * a3;
    const double c01 = a4 * a5 - a3 * a2, c02 = a3 * a5 - a1 * a4, c12 = a3 * a4 - a0 * a5;
    const double inv = 1.0 / (a0 * c00 + a3 * c01 + a4 * c02);
    const double p[6] = {c00 * inv, c11 * inv, c22 * inv, c01 * inv, c02 * inv, c12 * inv};
    const double A[6] = {a0, a1, a2, a3, a4, a5};
    // dsigma P, symmetrised (equal to P dsigma in exact arithmetic)
    auto m = [](const double* x, int i, int j) {
      const int idx[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
      return x[idx[i][j]];
    };
    double dp[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dp[i][j] = m(d, i, 0) * m(p, 0, j) + m(d, i, 1) * m(p, 1, j) + m(d, i, 2) * m(p, 2, j);
    const double q[6] = {dp[0][0], dp[1][1], dp[2][2], 0.5 * (dp[0][1] + dp[1][0]), 0.5 * (dp[0][2] + dp[2][0]),
                         0.5 * (dp[1][2] + dp[2][1])};
    for (int k = 0; k < 6; ++k) {
      pa[k * N + c] = A[k];
      pp[k * N + c] = p[k];
      pdp[k * N + c] = q[k];
    }
  }
}

ie_status ensure_precond(ie_ctx* c) {
  if (c->pre_p) return IE_OK;
  if (!c->contrast_set) return fail(c, IE_ERR_STATE, "preconditioner needs the contrast");
  const long long N = (long long)c->g.nx * c->g.ny * c->g.nz;
  IE_CUDA(c, cudaMalloc(&c->pre_p, 3 * 6 * N * sizeof(double)));
  c->pre_a = c->pre_p + 6 * N;
  c->pre_dp = c->pre_p + 12 * N;
  double* sbz = nullptr;
  std::vector<double> hsb;
  if (c->layered) {
    for (int k = 0; k < c->g.nz; ++k) hsb.push_back(sigma_b_at(c, k));
    IE_CUDA(c, cudaMalloc(&sbz, hsb.size() * sizeof(double)));
    IE_CUDA(c, cudaMemcpyAsync(sbz, hsb.data(), hsb.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  k_precond_build<<<grid_for(N, 256), 256, 0, c->stream>>>(c->dsig, c->pre_a, c->pre_p, c->pre_dp, N,
                                                           (long long)c->g.nx * c->g.ny, c->sigma_b, sbz);
  IE_CHECK_LAUNCH(c, "k_precond_build");
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(sbz);
  return IE_OK;
}

// y = M x per cell; M sym6 over the grid (strides cs, zs, ys), x and y compact over the box
__global__ void k_cellmat(double2* y, const double2* x, const double* __restrict__ M, int bx,
                          int by, int bz, long long cs, long long zs, long long ys) {
  const long long Nb = (long long)bx * by * bz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < Nb; i += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(i % bx), iy = (int)((i / bx) % by), iz = (int)(i / ((long long)bx * by));
    const double* m = M + iz * zs + iy * ys + ix;
    const double m0 = m[0], m1 = m[cs], m2 = m[2 * cs], m3 = m[3 * cs], m4 = m[4 * cs], m5 = m[5 * cs];
    const double2 x0 = x[i], x1 = x[Nb + i], x2 = x[2 * Nb + i];
    y[i] = make_double2(m0 * x0.x + m3 * x1.x + m4 * x2.x, m0 * x0.y + m3 * x1.y + m4 * x2.y);
    y[Nb + i] = make_double2(m3 * x0.x + m1 * x1.x + m5 * x2.x, m3 * x0.y + m1 * x1.y + m5 * x2.y);
    y[2 * Nb + i] = make_double2(m4 * x0.x + m5 * x1.x + m2 * x2.x, m4 * x0.y + m5 * x1.y + m2 * x2.y);
  }
}
void launch_cellmat(ie_ctx* c, double2* y, const double2* x, const double* M, int bx, int by, int bz, long long cs,
                    long long zs, long long ys) {
  const long long Nb = (long long)bx * by * bz;
  k_cellmat<<<grid_for(Nb, 256, 148 * 8), 256, 0, c->stream>>>(y, x, M, bx, by, bz, cs, zs, ys);
  c->launches++;
}

// per-system partial sums of |a - b|^2 -> part[sys][blk]; then fixed-order reduction
__global__ void __launch_bounds__(256) k_norm2_partial(const double2* __restrict__ a, const double2* __restrict__ b,
                                                       long long len, long long stride, double* __restrict__ part) {
  const int s = blockIdx.y;
  const double2* pa = a + s * stride;
  const double2* pb = b ? b + s * stride : nullptr;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    double2 v = pa[i];
    if (pb) v = csub(v, pb[i]);
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[s * gridDim.x + blockIdx.x] = red[0];
}
__global__ void k_sum_rows(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  const int s = blockIdx.x;
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) acc += part[s * nblk + i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[s] = red[0];
}

ie_status norms2(ie_ctx* c, const double2* a, const double2* b, int nsys, long long len, long long stride,
                 double* out_host) {
  const int nblk = 296;
  const size_t need = (size_t)nsys * nblk + nsys;
  if (c->d_red_cap * 2 < need) {
    if (c->d_red) cudaFree(c->d_red);
    c->d_red_cap = (need + 1) / 2 + 1024;
    IE_CUDA(c, cudaMalloc(&c->d_red, c->d_red_cap * sizeof(double2)));
  }
  double* part = (double*)c->d_red;
  double* res = part + (size_t)nsys * nblk;
  k_norm2_partial<<<dim3(nblk, nsys), 256, 0, c->stream>>>(a, b, len, stride, part);
  IE_CHECK_LAUNCH(c, "k_norm2_partial");
  k_sum_rows<<<nsys, 256, 0, c->stream>>>(part, nblk, res);
  IE_CHECK_LAUNCH(c, "k_sum_rows");
  IE_CUDA(c, cudaMemcpyAsync(out_host, res, nsys * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  return IE_OK;
}

}  // namespace ie
