// Complex128 Stockham FFT building blocks for sm_100a (device code only).
//
// A length-L line (L = 2^p, 2 <= L <= 1024) is transformed by T = L/V threads that each
// hold V = min(8, L) values in registers.  Each Stockham stage (Govindaraju et al. 2008
// formulation) reads R values at stride L/R, twiddles, does a radix-R DFT in registers and
// writes them to their auto-sorted positions; stages exchange through shared memory.
//  * The FIRST stage takes its inputs from registers (loaded by the caller straight from
//    global memory at positions  t + u*T + r*(L/R0)),
//  * the LAST stage leaves its outputs in registers at positions t + u*T + r*(L/Rlast),
// so global loads/stores are coalesced and no shared-memory staging is needed at either
// end.  Radix order "F" is 8,8,..,(4|4,4); order "B" is its reverse -- an inverse FFT run
// in order B starts on exactly the register positions a forward FFT in order F ends on,
// which lets the z-pass multiply the spectrum in registers (operator.cu, K-C).
// Twiddles come from per-stage tables tw[(r-1)*Ns + k] = exp(-2 pi i r k / (Ns R)) so
// that lanes with consecutive k read consecutive addresses.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

namespace ie {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// multiply by w4 = exp(DIR * i pi / 2) = DIR * i
template <int DIR>
__device__ __forceinline__ double2 mul_w4(double2 a) {
  return DIR > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
// multiply by w8 = exp(DIR * i pi / 4) = (1 + DIR i)/sqrt2
template <int DIR>
__device__ __forceinline__ double2 mul_w8(double2 a) {
  constexpr double s = 0.70710678118654752440084436210485;
  return DIR > 0 ? make_double2((a.x - a.y) * s, (a.y + a.x) * s) : make_double2((a.x + a.y) * s, (a.y - a.x) * s);
}
// multiply by w8^3 = exp(3 DIR i pi / 4) = (-1 + DIR i)/sqrt2
template <int DIR>
__device__ __forceinline__ double2 mul_w83(double2 a) {
  constexpr double s = 0.70710678118654752440084436210485;
  return DIR > 0 ? make_double2((-a.x - a.y) * s, (a.x - a.y) * s) : make_double2((a.y - a.x) * s, (-a.y - a.x) * s);
}

// In-place natural-order DFTs: X_k = sum_r v_r exp(DIR 2 pi i r k / R)
template <int DIR>
__device__ __forceinline__ void dft2(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
// HALF_IN: the upper half of the inputs is zero (not read); HALF_OUT: only the lower half of the
// outputs is produced (the others are left unspecified)
template <int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  if constexpr (HALF_IN) {  // v2 = v3 = 0
    const double2 a = v0, b = v1, wb = mul_w4<DIR>(b);
    v0 = cadd(a, b);
    v1 = cadd(a, wb);
    if constexpr (!HALF_OUT) {
      v2 = csub(a, b);
      v3 = csub(a, wb);
    }
  } else {
    double2 e0 = cadd(v0, v2), e1 = csub(v0, v2);
    double2 o0 = cadd(v1, v3), o1 = mul_w4<DIR>(csub(v1, v3));
    v0 = cadd(e0, o0);
    v1 = cadd(e1, o1);
    if constexpr (!HALF_OUT) {
      v2 = csub(e0, o0);
      v3 = csub(e1, o1);
    }
  }
}
template <int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dft4(double2* v) {
  dft4<DIR, HALF_IN, HALF_OUT>(v[0], v[1], v[2], v[3]);
}
template <int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dft8(double2* v) {
  double2 e0 = v[0], e1 = v[2], e2 = HALF_IN ? czero() : v[4], e3 = HALF_IN ? czero() : v[6];
  double2 o0 = v[1], o1 = v[3], o2 = HALF_IN ? czero() : v[5], o3 = HALF_IN ? czero() : v[7];
  dft4<DIR, HALF_IN>(e0, e1, e2, e3);  // (v0, v2, v4, v6): upper half v4, v6 zero when HALF_IN
  dft4<DIR, HALF_IN>(o0, o1, o2, o3);
  o1 = mul_w8<DIR>(o1);
  o2 = mul_w4<DIR>(o2);
  o3 = mul_w83<DIR>(o3);
  v[0] = cadd(e0, o0);
  v[1] = cadd(e1, o1);
  v[2] = cadd(e2, o2);
  v[3] = cadd(e3, o3);
  if constexpr (!HALF_OUT) {
    v[4] = csub(e0, o0);
    v[5] = csub(e1, o1);
    v[6] = csub(e2, o2);
    v[7] = csub(e3, o3);
  }
}
// multiply by w16 = exp(DIR i pi/8) and w16^3 = exp(3 DIR i pi/8)
template <int DIR>
__device__ __forceinline__ double2 mul_w16(double2 a) {
  constexpr double c = 0.92387953251128675612818318939678829, s = DIR * 0.38268343236508977172845998403039887;
  return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
}
template <int DIR>
__device__ __forceinline__ double2 mul_w163(double2 a) {
  constexpr double c = 0.38268343236508977172845998403039887, s = DIR * 0.92387953251128675612818318939678829;
  return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
}

// 16-point DFT, natural order, as 4 x 4 (n = 4 n1 + n2, k = k1 + 4 k2).
// HALF_IN: v[8..15] are zero and not read (the zero-padded upper half of a forward pass);
// HALF_OUT: only X[0..7] are produced (the cropped lower half of an inverse pass).
template <int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dft16(double2* v) {
  double2 a[4][4];  // a[n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    if constexpr (HALF_IN) {
      const double2 x0 = v[n2], x1 = v[4 + n2], w = mul_w4<DIR>(x1);
      a[n2][0] = cadd(x0, x1);
      a[n2][1] = cadd(x0, w);
      a[n2][2] = csub(x0, x1);
      a[n2][3] = csub(x0, w);
    } else {
      a[n2][0] = v[n2];
      a[n2][1] = v[4 + n2];
      a[n2][2] = v[8 + n2];
      a[n2][3] = v[12 + n2];
      dft4<DIR>(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
    }
  }
  a[1][1] = mul_w16<DIR>(a[1][1]);
  a[1][2] = mul_w8<DIR>(a[1][2]);
  a[1][3] = mul_w163<DIR>(a[1][3]);
  a[2][1] = mul_w8<DIR>(a[2][1]);
  a[2][2] = mul_w4<DIR>(a[2][2]);
  a[2][3] = mul_w83<DIR>(a[2][3]);
  a[3][1] = mul_w163<DIR>(a[3][1]);
  a[3][2] = mul_w83<DIR>(a[3][2]);
  {
    const double2 m = mul_w16<DIR>(a[3][3]);  // w16^9 = -w16
    a[3][3] = make_double2(-m.x, -m.y);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    const double2 e0 = cadd(a[0][k1], a[2][k1]), e1 = csub(a[0][k1], a[2][k1]);
    const double2 o0 = cadd(a[1][k1], a[3][k1]), o1 = mul_w4<DIR>(csub(a[1][k1], a[3][k1]));
    v[k1] = cadd(e0, o0);
    v[k1 + 4] = cadd(e1, o1);
    if constexpr (!HALF_OUT) {
      v[k1 + 8] = csub(e0, o0);
      v[k1 + 12] = csub(e1, o1);
    }
  }
}

// cos / sin of k pi / 8, k = 0 .. 15
__host__ __device__ constexpr double cos_pi8(int k) {
  constexpr double c[16] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                            0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                            -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
                            0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};
  return c[k & 15];
}
__host__ __device__ constexpr double sin_pi8(int k) { return cos_pi8(k - 4); }

// p = a + T b, m = a - T b for the constant T = exp(DIR i pi E / 8), FMA-shaped: T b = c (b (1 + i tau))
// (|cos| >= |sin|) or s (b (cot + i)) (otherwise), so the product folds into the butterfly's
// additions (6 FP64 instructions for a general T instead of 4 for the product + 4 for the
// additions; 4 for T = +-1, +-i; 6 for the odd multiples of pi/4). ONLY_P: p alone.
template <int DIR, int E, bool ONLY_P = false>
__device__ __forceinline__ void bfly_rot(const double2 a, const double2 b, double2& p, double2& m) {
  constexpr int e = ((E % 16) + 16) % 16;
  constexpr double c = cos_pi8(e), sn = DIR * sin_pi8(e);
  if constexpr (e == 0 || e == 8) {
    const double2 tb = e == 0 ? b : make_double2(-b.x, -b.y);
    p = cadd(a, tb);
    if constexpr (!ONLY_P) m = csub(a, tb);
  } else if constexpr (e == 4 || e == 12) {
    const double2 tb = ((e == 4) == (DIR > 0)) ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
    p = cadd(a, tb);
    if constexpr (!ONLY_P) m = csub(a, tb);
  } else if constexpr ((e & 3) == 2) {  // T = h (sc + i ss), h = 1/sqrt2, sc, ss = +-1
    constexpr double h = 0.70710678118654752440;
    constexpr bool pc = c > 0, ps = sn > 0;
    const double yx = pc ? (ps ? b.x - b.y : b.x + b.y) : (ps ? -b.x - b.y : b.y - b.x);
    const double yy = pc ? (ps ? b.y + b.x : b.y - b.x) : (ps ? b.x - b.y : -b.y - b.x);
    p = make_double2(fma(h, yx, a.x), fma(h, yy, a.y));
    if constexpr (!ONLY_P) m = make_double2(fma(-h, yx, a.x), fma(-h, yy, a.y));
  } else if constexpr ((c > 0 ? c : -c) >= (sn > 0 ? sn : -sn)) {
    constexpr double tau = sn / c;
    const double yx = fma(-tau, b.y, b.x), yy = fma(tau, b.x, b.y);
    p = make_double2(fma(c, yx, a.x), fma(c, yy, a.y));
    if constexpr (!ONLY_P) m = make_double2(fma(-c, yx, a.x), fma(-c, yy, a.y));
  } else {
    constexpr double kap = c / sn;
    const double yx = fma(kap, b.x, -b.y), yy = fma(kap, b.y, b.x);
    p = make_double2(fma(sn, yx, a.x), fma(sn, yy, a.y));
    if constexpr (!ONLY_P) m = make_double2(fma(-sn, yx, a.x), fma(-sn, yy, a.y));
  }
}

// dft16 with the 4 x 4 split's inner twiddles w16^(n2 k1) folded into the second layer's
// butterflies (bfly_rot): the same transform with 12 fewer FP64 instructions (148 vs 160 full)
template <int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dft16f(double2* v) {
  double2 a[4][4];  // a[n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    if constexpr (HALF_IN) {
      const double2 x0 = v[n2], x1 = v[4 + n2], w = mul_w4<DIR>(x1);
      a[n2][0] = cadd(x0, x1);
      a[n2][1] = cadd(x0, w);
      a[n2][2] = csub(x0, x1);
      a[n2][3] = csub(x0, w);
    } else {
      a[n2][0] = v[n2];
      a[n2][1] = v[4 + n2];
      a[n2][2] = v[8 + n2];
      a[n2][3] = v[12 + n2];
      dft4<DIR>(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
    }
  }
  // X[k1 + 4 k2] = sum_n2 a[n2][k1] T^n2 (DIR i)^(n2 k2), T = w16^k1:
  //   e0/e1 = a0 +- T^2 a2, p/m = a1 +- T^2 a3, X[k1] / X[k1+8] = e0 +- T p, X[k1+4] / X[k1+12] = e1 +- (DIR i T) m
  auto col = [&](auto k1c) {
    constexpr int k1 = decltype(k1c)::value;
    double2 e0, e1, p, m;
    bfly_rot<DIR, 2 * k1>(a[0][k1], a[2][k1], e0, e1);
    bfly_rot<DIR, 2 * k1>(a[1][k1], a[3][k1], p, m);
    bfly_rot<DIR, k1, HALF_OUT>(e0, p, v[k1], v[k1 + 8]);
    bfly_rot<DIR, k1 + 4, HALF_OUT>(e1, m, v[k1 + 4], v[k1 + 12]);
  };
  col(std::integral_constant<int, 0>{});
  col(std::integral_constant<int, 1>{});
  col(std::integral_constant<int, 2>{});
  col(std::integral_constant<int, 3>{});
}

template <int R, int DIR, bool HALF_IN = false, bool HALF_OUT = false>
__device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 2) dft2<DIR>(v);
  else if constexpr (R == 4) dft4<DIR, HALF_IN, HALF_OUT>(v);
  else if constexpr (R == 8) dft8<DIR, HALF_IN, HALF_OUT>(v);
  else dft16<DIR, HALF_IN, HALF_OUT>(v);
}

// ------------------------------------------------------------------------ plans
__host__ __device__ constexpr int log2c(int L) { return L <= 1 ? 0 : 1 + log2c(L / 2); }

template <int L>
struct FftPlan {
  static constexpr int P = log2c(L);
  static constexpr int NST = (P <= 3) ? 1 : (P + 2) / 3;
  static constexpr int V = L < 8 ? L : 8;
  static constexpr int T = L / V;
  // forward ("F") radix order
  __host__ __device__ static constexpr int radixF(int s) {
    return (P <= 3) ? L : (s < ((P % 3 == 0) ? P / 3 : (P % 3 == 2) ? P / 3 : P / 3 - 1) ? 8 : 4);
  }
  __host__ __device__ static constexpr int radix(int s, bool rev) { return rev ? radixF(NST - 1 - s) : radixF(s); }
  __host__ __device__ static constexpr int ns(int s, bool rev) { return s == 0 ? 1 : ns(s - 1, rev) * radix(s - 1, rev); }
  // twiddle table offset of stage s (s >= 1): sum over earlier stages of (R-1)*Ns
  __host__ __device__ static constexpr int twoff(int s, bool rev) {
    return s <= 1 ? 0 : twoff(s - 1, rev) + (radix(s - 1, rev) - 1) * ns(s - 1, rev);
  }
  __host__ __device__ static constexpr int twsize(bool rev) { return twoff(NST, rev); }
};

// shared-memory index for element i of a column c among W interleaved columns, padded by
// one element per 8 so that stride-8 (128-byte) lane patterns do not bank-conflict.
struct SIdx {
  int base, W, c;
  __device__ __forceinline__ int operator()(int i) const {
    int a = i * W + c;
    return base + a + (a >> 3);
  }
};
__host__ __device__ constexpr int padded(int n) { return n + (n >> 3); }

// Transform NL lines held by this thread (v[l][0..V)) through all stages.
//   entry: v[l][u*R0 + r] = x_l[t + u*T + r*L/R0]            (R0 = first radix)
//   exit : v[l][u*RL + r] = X_l[t + u*T + r*L/RL]            (RL = last radix)
// sm + idx(l)(i): shared-memory slot of element i of line l.  tw: twiddle table of this
// (L, order).  need_sync_first: a __syncthreads() before the first shared write (when the
// regions were read just before).  All threads of the CTA must call this (barriers).
template <int L, bool REV, int DIR, int NL, int S, bool HOUT = false, class IdxF>
__device__ __forceinline__ void fft_stage(double2 (&v)[NL][FftPlan<L>::V], double2* sm, IdxF idx, int t,
                                          const double2* __restrict__ tw) {
  using P = FftPlan<L>;
  constexpr int V = P::V, T = P::T, NST = P::NST;
  constexpr int R = P::radix(S, REV);
  constexpr int Ns = P::ns(S, REV);
  constexpr int U = V / R;
  const double2* tws = tw + P::twoff(S, REV);
#pragma unroll
  for (int l = 0; l < NL; ++l)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u * T;
#pragma unroll
      for (int r = 0; r < R; ++r) v[l][u * R + r] = sm[idx(l)(j + r * (L / R))];
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = t + u * T;
    const int k = j & (Ns - 1);
    // stage twiddles w^r, w = exp(-2 pi i k / (Ns R)): R = 8 from two loaded powers (w, w^4)
    // and five complex multiplies instead of seven loads; R = 4 from w alone
    double2 w[R];
    if constexpr (R == 8) {
      w[1] = __ldg(&tws[k]);
      w[4] = __ldg(&tws[3 * Ns + k]);
      w[2] = cmul(w[1], w[1]);
      w[3] = cmul(w[2], w[1]);
      w[5] = cmul(w[4], w[1]);
      w[6] = cmul(w[4], w[2]);
      w[7] = cmul(w[4], w[3]);
    } else if constexpr (R == 4) {
      w[1] = __ldg(&tws[k]);
      w[2] = cmul(w[1], w[1]);
      w[3] = cmul(w[2], w[1]);
    } else {
#pragma unroll
      for (int r = 1; r < R; ++r) w[r] = __ldg(&tws[(r - 1) * Ns + k]);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
#pragma unroll
      for (int r = 1; r < R; ++r)
        v[l][u * R + r] = (DIR < 0) ? cmul(v[l][u * R + r], w[r]) : cmulc(v[l][u * R + r], w[r]);
      dftR<R, DIR, false, HOUT && S == NST - 1>(&v[l][u * R]);
    }
  }
  if constexpr (S < NST - 1) {
    __syncthreads();
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t + u * T;
        const int k = j & (Ns - 1);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) sm[idx(l)(base + r * Ns)] = v[l][u * R + r];
      }
    __syncthreads();
    fft_stage<L, REV, DIR, NL, S + 1, HOUT>(v, sm, idx, t, tw);
  }
}

// HIN: the upper half of every first-stage radix group is zero (zero-padded forward input);
// HOUT: only the lower half of every last-stage radix group is needed (cropped inverse output)
template <int L, bool REV, int DIR, int NL, bool HIN = false, bool HOUT = false, class IdxF>
__device__ __forceinline__ void fft_run(double2 (&v)[NL][FftPlan<L>::V], double2* sm, IdxF idx, int t,
                                        const double2* __restrict__ tw, bool need_sync_first) {
  using P = FftPlan<L>;
  constexpr int V = P::V, T = P::T, NST = P::NST;
  constexpr int R0 = P::radix(0, REV);
#pragma unroll
  for (int l = 0; l < NL; ++l)
#pragma unroll
    for (int u = 0; u < V / R0; ++u) dftR<R0, DIR, HIN, HOUT && NST == 1>(&v[l][u * R0]);
  if constexpr (NST > 1) {
    if (need_sync_first) __syncthreads();
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int u = 0; u < V / R0; ++u) {
        const int j = t + u * T;
#pragma unroll
        for (int r = 0; r < R0; ++r) sm[idx(l)(j * R0 + r)] = v[l][u * R0 + r];
      }
    __syncthreads();
    fft_stage<L, REV, DIR, NL, 1, HOUT>(v, sm, idx, t, tw);
  }
}

}  // namespace ie
