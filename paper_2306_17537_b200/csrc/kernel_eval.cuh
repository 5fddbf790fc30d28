// The discrete homogeneous kernel K(d) = G^E(d h) dv (Eq. 5 at centroid offsets, midpoint
// rule) with the equivolume-sphere self term at d = 0 (reading R3).  Shared by the
// Green-spectrum setup (green.cu) and the degenerate layered table (layered.cu).
#pragma once
#include <cuda_runtime.h>

#include "ie_internal.h"

namespace ie {

struct GreenArgs {
  int nx, ny, nz;
  double dx, dy, dz, dv;
  double k0r, k0i, sigma_b;
  double selfr, selfi;
};

__device__ __forceinline__ double2 cexp_i(double2 z) {  // exp(i z)
  const double m = exp(-z.y);
  double s, c;
  sincos(z.x, &s, &c);
  return make_double2(m * c, m * s);
}

// component comp in 0..5 = (xx, yy, zz, xy, xz, yz) of K at lattice offset (dxi, dyi, dzi)
__device__ __forceinline__ double2 kernel_sample(const GreenArgs& a, int dxi, int dyi, int dzi, int comp) {
  if (dxi == 0 && dyi == 0 && dzi == 0) return comp < 3 ? make_double2(a.selfr, a.selfi) : make_double2(0.0, 0.0);
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
  switch (comp) {
    case 0: hp = hx; hq = hx; break;
    case 1: hp = hy; hq = hy; break;
    case 2: hp = hz; hq = hz; break;
    case 3: hp = hx; hq = hy; break;
    case 4: hp = hx; hq = hz; break;
    default: hp = hy; hq = hz; break;
  }
  double2 coef = make_double2(be.x * hp * hq, be.y * hp * hq);
  if (comp < 3) coef = make_double2(coef.x + al.x, coef.y + al.y);
  const double s = a.dv / a.sigma_b;
  return make_double2((coef.x * g.x - coef.y * g.y) * s, (coef.x * g.y + coef.y * g.x) * s);
}

GreenArgs green_args(const ie_ctx* c, int nx, int ny, int nz);

}  // namespace ie
