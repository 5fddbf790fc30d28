// A3L: the IE operator over a horizontally layered background (
// DESIGN.md readings R17-R19).  The kernel is translation invariant in x and y only:
//     (G J)_p(i,j,k) = sum_{q,i',j',k'} T_pq(i-i', j-j'; k, k') J_q(i',j',k')
// with T a table of kernel samples supplied by the caller (host, complex128, quadrant of
// non-negative offsets [9][nz][nz][ny][nx], mirror rules sx = (-1,1,1), sy = (1,-1,1)) or,
// for format 2, the degenerate equal-layer table built here from the homogeneous kernel.
//
// Setup (per domain shape and z-range, like the homogeneous Green spectrum): every
// (p,q,k,k') plane is circulant-embedded on (2ny, 2nx), FFT'd in x and y, and packed to the
// quadrant of horizontal wavenumbers (ix <= nx, iy <= ny) as one (3nz x 3nz) matrix per
// wavenumber: mhat[(iy (nx+1) + ix)][(q nz + k')][(p nz + k)], scaled 1/(4 nx ny).
//
// Apply: K-A, K-B (x, y forward FFTs) and K-D, K-E (inverse) are the homogeneous kernels;
// the z-pass K-C is replaced by K-C' (k_zlayer): for each quadrant wavenumber the up-to-4
// mirror columns (+-kx, +-ky) of every right-hand side are contracted with the one matrix
// M (the full-spectrum matrix at a mirrored wavenumber is D M D, D = diag(sx, sy, 1)).
#include <math.h>

#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "bulk_copy.cuh"
#include "fft_core.cuh"
#include "ie_internal.h"
#include "pdl.cuh"
#include "kernel_eval.cuh"

namespace ie {

double sigma_b_at(const ie_ctx* c, int k) {
  if (!c->layered || c->lay_sigma.size() <= 1) return c->sigma_b;
  const double z = c->g.origin[2] + k * c->g.dz;
  size_t l = 0;
  while (l < c->lay_z.size() && z >= c->lay_z[l]) ++l;  // layer l: z_iface[l-1] <= z < z_iface[l]
  return c->lay_sigma[l];
}

// ------------------------------------------------------------------ table (format 2)
// degenerate equal-layer table: T_pq(di, dj; k, k') = K_pq(di, dj, k - k')
__global__ void k_table_homog(double2* __restrict__ T, GreenArgs a) {
  const long long nx = a.nx, ny = a.ny, nz = a.nz;
  const long long total = 9 * nz * nz * ny * nx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int di = (int)(e % nx), dj = (int)((e / nx) % ny);
    const int kp = (int)((e / (nx * ny)) % nz), k = (int)((e / (nx * ny * nz)) % nz);
    const int pq = (int)(e / (nx * ny * nz * nz)), pp = pq / 3, qq = pq % 3;
    const int comp = (pp == qq) ? pp : (pp + qq == 1 ? 3 : (pp + qq == 2 ? 4 : 5));
    T[e] = kernel_sample(a, di, dj, k - kp, comp);
  }
}

ie_status build_layer_table(ie_ctx* c, const void* host_table) {
  const long long nx = c->g.nx, ny = c->g.ny, nz = c->g.nz;
  const size_t bytes = (size_t)9 * nz * nz * ny * nx * sizeof(double2);
  IE_CUDA(c, cudaMalloc(&c->tab, bytes));
  if (host_table) {
    IE_CUDA(c, cudaMemcpyAsync(c->tab, host_table, bytes, cudaMemcpyHostToDevice, c->stream));
  } else {
    const GreenArgs a = green_args(c, (int)nx, (int)ny, (int)nz);
    k_table_homog<<<2368, 256, 0, c->stream>>>(c->tab, a);
    IE_CHECK_LAUNCH(c, "k_table_homog");
  }
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  return IE_OK;
}

// ------------------------------------------------------------------ spectra
// plane pl (of a chunk starting at plane p0) = (pq, k, k') over the box's (bz x bz) layers
__global__ void k_layer_embed(const double2* __restrict__ T, double2* __restrict__ C, int NX, int NY, int NZ,
                              int bx, int by, int bz, int k0, long long p0, int nplanes) {
  const long long Lx = 2 * bx, Ly = 2 * by, per = Lx * Ly, total = per * nplanes;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long pl = p0 + e / per;
    const int u = (int)(e % Lx), v = (int)((e / Lx) % Ly);
    const int kp = (int)(pl % bz), k = (int)((pl / bz) % bz), pq = (int)(pl / ((long long)bz * bz));
    double2 val = make_double2(0.0, 0.0);
    if (u != bx && v != by) {
      const int di = u < bx ? u : (int)(Lx - u), dj = v < by ? v : (int)(Ly - v);  // |offset|
      const int pp = pq / 3, qq = pq % 3;
      const bool oddx = (pp == 0) != (qq == 0), oddy = (pp == 1) != (qq == 1);  // sx_p sx_q, sy_p sy_q = -1
      double s = 1.0;
      if (u > bx && oddx) s = -s;  // di < 0
      if (v > by && oddy) s = -s;  // dj < 0
      if ((di == 0 && oddx) || (dj == 0 && oddy)) s = 0.0;  // the rules force 0 at zero offset
      const double2 t = T[((((long long)pq * NZ + (k0 + k)) * NZ + (k0 + kp)) * NY + dj) * NX + di];
      val = make_double2(s * t.x, s * t.y);
    }
    C[e] = val;
  }
}

__global__ void k_layer_pack(const double2* __restrict__ C, double2* __restrict__ M, int bx, int by, int bz,
                             long long p0, int nplanes, double scale) {
  const long long Ox = bx + 1, Oy = by + 1, per = Ox * Oy, total = per * nplanes;
  const long long Lx = 2 * bx, Ly = 2 * by, R = 3LL * bz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long pl = p0 + e / per, loc = e / per;
    const int ix = (int)(e % Ox), iy = (int)((e / Ox) % Oy);
    const int kp = (int)(pl % bz), k = (int)((pl / bz) % bz), pq = (int)(pl / ((long long)bz * bz));
    const int pp = pq / 3, qq = pq % 3;
    const double2 v = C[(loc * Ly + iy) * Lx + ix];
    M[((long long)iy * Ox + ix) * R * R + (qq * bz + kp) * R + (pp * bz + k)] = make_double2(v.x * scale, v.y * scale);
  }
}

ie_status build_layer_spec(ie_ctx* c, int bx, int by, int bz, int k0, GreenSpec* out) {
  if (!c->tab) return fail(c, IE_ERR_STATE, "layered context without a table");
  const long long Lx = 2 * bx, Ly = 2 * by, R = 3LL * bz;
  const long long planes = 9LL * bz * bz;
  out->nx = bx;
  out->ny = by;
  out->nz = bz;
  out->k0 = k0;
  out->oct = nullptr;
  IE_CUDA(c, cudaMalloc(&out->mhat, (size_t)(bx + 1) * (by + 1) * R * R * sizeof(double2)));
  // planes per chunk: about 512 MB of embedded planes at a time
  const long long per = Lx * Ly;
  const long long chunk = std::max(1LL, std::min(planes, (512LL << 20) / (per * (long long)sizeof(double2))));
  double2* C = nullptr;
  IE_CUDA(c, cudaMalloc(&C, (size_t)chunk * per * sizeof(double2)));
  const double scale = 1.0 / (double)(Lx * Ly);
  cudaError_t e = cudaSuccess;
  for (long long p0 = 0; p0 < planes && e == cudaSuccess; p0 += chunk) {
    const int np = (int)std::min(chunk, planes - p0);
    k_layer_embed<<<2368, 256, 0, c->stream>>>(c->tab, C, c->g.nx, c->g.ny, c->g.nz, bx, by, bz, k0, p0, np);
    c->launches++;
    e = cudaGetLastError();
    if (!e) e = fft_axis((int)Lx, C, 1, (long long)np * Ly, c->tw.get((int)Lx, 0), c->stream);
    if (!e) e = fft_axis((int)Ly, C, Lx, np, c->tw.get((int)Ly, 0), c->stream);
    c->launches += 2;
    if (!e) {
      k_layer_pack<<<2368, 256, 0, c->stream>>>(C, out->mhat, bx, by, bz, p0, np, scale);
      c->launches++;
      e = cudaGetLastError();
    }
  }
  if (!e) e = cudaStreamSynchronize(c->stream);
  cudaFree(C);
  if (e) {
    cudaFree(out->mhat);
    out->mhat = nullptr;
    return cuda_fail(c, e, "layered spectrum setup");
  }
  return IE_OK;
}

// ------------------------------------------------------------------ K-C'
// One CTA per quadrant wavenumber (ix, iy).  Its mirror columns kx in {ix, 2nx-ix},
// ky in {iy, 2ny-iy} (1, 2 or 4 distinct) of NI right-hand sides share the matrix M(ix,iy):
//   Y(col) = D_col M D_col X(col),  D = diag(sx, sy, 1) of the column's mirror signs.
// X (3nz x 4NI, signs applied) sits in shared memory; each thread owns output rows (p,k) and
// streams its column of M (consecutive rows across threads: coalesced 16-byte loads), only
// over the source rows k' in [sz0, sz1) (a source-restricted apply reads less of M).
template <int NI>
__global__ void __launch_bounds__(256) k_zlayer(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  constexpr int NS = 4 * NI;  // column slots: (cy*2 + cx)*NI + item
  extern __shared__ __align__(16) double2 xs[];
  const int nx = p.nx, ny = p.ny, nz = p.nz, Lx = 2 * nx, Ly = 2 * ny, R = 3 * nz;
  const int ixy = blockIdx.x, ix = ixy % (nx + 1), iy = ixy / (nx + 1);
  const int kxs[2] = {ix, Lx - ix}, kys[2] = {iy, Ly - iy};
  const int nkx = (ix == 0 || ix == nx) ? 1 : 2, nky = (iy == 0 || iy == ny) ? 1 : 2;
  const long long cs = (long long)nz * Ly * Lx, zs = (long long)Ly * Lx;
  const int z0 = p.items[0].sz0, z1 = p.items[0].sz1;
  for (int e = threadIdx.x; e < R * NS; e += blockDim.x) {
    const int slot = e % NS, row = e / NS, q = row / nz, kp = row % nz;
    const int item = slot % NI, cc = slot / NI, cx = cc & 1, cy = cc >> 1;
    double2 v = czero();
    if (item < p.n_items && cx < nkx && cy < nky && kp >= z0 && kp < z1) {
      v = p.X2[(long long)item * 3 * cs + q * cs + kp * zs + (long long)kys[cy] * Lx + kxs[cx]];
      if ((q == 0 && cx == 1) || (q == 1 && cy == 1)) v = make_double2(-v.x, -v.y);
    }
    xs[e] = v;
  }
  __syncthreads();
  const double2* M = p.mhat + (long long)ixy * R * R;
  for (int pk = threadIdx.x; pk < R; pk += blockDim.x) {
    double2 acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = czero();
    for (int q = 0; q < 3; ++q) {
      const double2* Mq = M + (long long)(q * nz) * R + pk;
      const double2* xq = xs + (q * nz) * NS;
#pragma unroll 4
      for (int kp = z0; kp < z1; ++kp) {
        const double2 m = __ldg(Mq + (long long)kp * R);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const double2 x = xq[kp * NS + s];
          acc[s].x = fma(m.x, x.x, fma(-m.y, x.y, acc[s].x));
          acc[s].y = fma(m.x, x.y, fma(m.y, x.x, acc[s].y));
        }
      }
    }
    const int pp = pk / nz, k = pk % nz;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int item = s % NI, cc = s / NI, cx = cc & 1, cy = cc >> 1;
      if (item < p.n_items && cx < nkx && cy < nky) {
        double2 v = acc[s];
        if ((pp == 0 && cx == 1) || (pp == 1 && cy == 1)) v = make_double2(-v.x, -v.y);
        p.X2[(long long)item * 3 * cs + pp * cs + k * zs + (long long)kys[cy] * Lx + kxs[cx]] = v;
      }
    }
  }
  pdl_trigger_late();
}

// The same contraction on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64) when the
// right-hand sides make it a real contraction (NI >= 2: 4 NI >= 8 columns, one n-tile per 8)
// and 3nz is a multiple of 8.  A = M (rows (p,k), cols (q,k')), B = X (rows (q,k'), cols =
// column slots), complex as four real MMAs per (k-step, n-tile).  Fragments (PTX m8n8k4 f64):
// lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}].  Each warp owns 8-row tiles
// and streams its rows of M with 16-byte loads (8 consecutive rows x 4 k: 128-byte segments).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NI>
__global__ void __launch_bounds__(256) k_zlayer_mma(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  constexpr int NS = 4 * NI, NT = (NS + 7) / 8, NSP = NT * 8;
  extern __shared__ __align__(16) double2 xs[];  // [R][NSP], signs applied, zero padded
  const int nx = p.nx, ny = p.ny, nz = p.nz, Lx = 2 * nx, Ly = 2 * ny, R = 3 * nz;
  const int ixy = blockIdx.x, ix = ixy % (nx + 1), iy = ixy / (nx + 1);
  const int kxs[2] = {ix, Lx - ix}, kys[2] = {iy, Ly - iy};
  const int nkx = (ix == 0 || ix == nx) ? 1 : 2, nky = (iy == 0 || iy == ny) ? 1 : 2;
  const long long cs = (long long)nz * Ly * Lx, zs = (long long)Ly * Lx;
  const int z0 = p.items[0].sz0, z1 = p.items[0].sz1;
  for (int e = threadIdx.x; e < R * NSP; e += blockDim.x) {
    const int slot = e % NSP, row = e / NSP, q = row / nz, kp = row % nz;
    const int item = slot % NI, cc = slot / NI, cx = cc & 1, cy = cc >> 1;
    double2 v = czero();
    if (slot < NS && item < p.n_items && cx < nkx && cy < nky && kp >= z0 && kp < z1) {
      v = p.X2[(long long)item * 3 * cs + q * cs + kp * zs + (long long)kys[cy] * Lx + kxs[cx]];
      if ((q == 0 && cx == 1) || (q == 1 && cy == 1)) v = make_double2(-v.x, -v.y);
    }
    xs[e] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;  // A[ar][ac], B[ac][ar], C[ar][2 ac + j]
  const double2* M = p.mhat + (long long)ixy * R * R;
  for (int rt = warp; rt < R / 8; rt += nwarps) {
    const int r0 = rt * 8;
    double cr[NT][2], ci[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) cr[t][0] = cr[t][1] = ci[t][0] = ci[t][1] = 0.0;
    const double2* Ma = M + (long long)ac * R + r0 + ar;
#pragma unroll 4
    for (int k0 = 0; k0 < R; k0 += 4) {
      const double2 a = __ldg(Ma + (long long)k0 * R);
      const double nai = -a.y;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double2 b = xs[(k0 + ac) * NSP + t * 8 + ar];
        dmma(cr[t][0], cr[t][1], a.x, b.x);
        dmma(cr[t][0], cr[t][1], nai, b.y);
        dmma(ci[t][0], ci[t][1], a.x, b.y);
        dmma(ci[t][0], ci[t][1], a.y, b.x);
      }
    }
    const int pk = r0 + ar, pp = pk / nz, k = pk % nz;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int s = t * 8 + 2 * ac + j;
        const int item = s % NI, cc = s / NI, cx = cc & 1, cy = cc >> 1;
        if (s < NS && item < p.n_items && cx < nkx && cy < nky) {
          double2 v = make_double2(cr[t][j], ci[t][j]);
          if ((pp == 0 && cx == 1) || (pp == 1 && cy == 1)) v = make_double2(-v.x, -v.y);
          p.X2[(long long)item * 3 * cs + pp * cs + k * zs + (long long)kys[cy] * Lx + kxs[cx]] = v;
        }
      }
  }
  pdl_trigger_late();
}

// Warp-specialised version: a producer warp streams M(ix,iy) into a 2-stage shared ring with
// bulk asynchronous copies (TMA bulk mode, one 8-row chunk = 8*3nz*16 contiguous bytes per
// copy, completion on mbarriers); 8 consumer warps feed the DMMA tensor cores from shared
// memory and release each stage through an "empty" mbarrier, so HBM streaming is decoupled
// from the tensor-core work.  Complex arithmetic without padding: B is X viewed as real
// columns (Re X_s, Im X_s interleaved, 2*4NI columns = NI n-tiles of 8), and per k-step
// C1 += Re(M) B, C2 += Im(M) B; a lane's C pair (2j, 2j+1) is (Re X_s, Im X_s) of one slot,
// so Y_s = (C1[2s] - C2[2s+1]) + i (C1[2s+1] + C2[2s]) in registers.
template <int NI, int RT>
__global__ void __launch_bounds__(288, 2) k_zlayer_tma(const __grid_constant__ ApplyParams p) {
  pdl_wait();
  constexpr int NS = 4 * NI, NT = NI;      // slots; real columns 2 NS = 8 NI: NI n-tiles
  // k-rows per chunk, ring stages (3 for one RHS, where the consumers outpace a 2-deep ring;
  // 2 otherwise: c3h 1 RHS 0.517 -> 0.506 ms, 3 RHS 0.735 vs 0.760 ms), consumer warps
  constexpr int KC = 8, NST = NI == 1 ? 3 : 2, NCW = 8;
  extern __shared__ __align__(128) double2 smem[];
  const int nx = p.nx, ny = p.ny, nz = p.nz, Lx = 2 * nx, Ly = 2 * ny, R = 3 * nz;
  double2* xs = smem;                     // [R][NS] complex = [R][2NS] real
  const double* xd = reinterpret_cast<const double*>(xs);
  double2* ring = smem + R * NS;          // [NST][KC][R]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NST * KC * R);
  uint64_t* empty = full + NST;
  const int ixy = blockIdx.x, ix = ixy % (nx + 1), iy = ixy / (nx + 1);
  const int kxs[2] = {ix, Lx - ix}, kys[2] = {iy, Ly - iy};
  const int nkx = (ix == 0 || ix == nx) ? 1 : 2, nky = (iy == 0 || iy == ny) ? 1 : 2;
  const long long cs = (long long)nz * Ly * Lx, zs = (long long)Ly * Lx;
  const int z0 = p.items[0].sz0, z1 = p.items[0].sz1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = R / KC;
  const double2* M = p.mhat + (long long)ixy * R * R;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
  }
  __syncthreads();
  // a chunk of KC source rows (q nz + k', one q: nz is a multiple of KC) matters only if its k'
  // range meets the items' source range [z0, z1) (z-restricted Gauss-Seidel couplings); the
  // producer and the consumers skip the same chunks
  auto active = [&](int ch) {
    const int kp0 = (ch * KC) % nz;
    return kp0 + KC > z0 && kp0 < z1;
  };
  if (warp == NCW) {  // ---- producer
    if (lane == 0) {
      for (int ch = 0, a = 0; ch < nchunks; ++ch) {
        if (!active(ch)) continue;
        const int st = a % NST;
        if (a >= NST) mbar_wait(&empty[st], ((a / NST) - 1) & 1);
        const uint32_t bytes = (uint32_t)(KC * R * sizeof(double2));
        mbar_arrive_expect_tx(&full[st], bytes);
        bulk_g2s(ring + st * KC * R, M + (long long)ch * KC * R, bytes, &full[st]);
        ++a;
      }
    }
    return;
  }
  // ---- consumers: stage X (signs applied), then the DMMA loop.  The gathers (one 16-byte
  // element per (row, slot), scattered over the four mirror columns) go out in batches of BT
  // loads per thread before any is used, so their latencies overlap
  constexpr int BT = 6;
  for (int e0 = threadIdx.x; e0 < R * NS; e0 += BT * NCW * 32) {
    double2 v[BT];
    bool neg[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int e = e0 + b * NCW * 32;
      v[b] = czero();
      neg[b] = false;
      if (e < R * NS) {
        const int slot = e % NS, row = e / NS, q = row / nz, kp = row % nz;
        const int item = slot % NI, cc = slot / NI, cx = cc & 1, cy = cc >> 1;
        if (item < p.n_items && cx < nkx && cy < nky && kp >= z0 && kp < z1) {
          v[b] = __ldg(&p.X2[(long long)item * 3 * cs + q * cs + kp * zs + (long long)kys[cy] * Lx + kxs[cx]]);
          neg[b] = (q == 0 && cx == 1) || (q == 1 && cy == 1);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int e = e0 + b * NCW * 32;
      if (e < R * NS) xs[e] = neg[b] ? make_double2(-v[b].x, -v[b].y) : v[b];
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32));  // consumers only
  const int ar = lane >> 2, ac = lane & 3;
  double c1[RT][NT][2], c2[RT][NT][2];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int t = 0; t < NT; ++t) c1[r][t][0] = c1[r][t][1] = c2[r][t][0] = c2[r][t][1] = 0.0;
  for (int ch = 0, ach = 0; ch < nchunks; ++ch) {
    if (!active(ch)) continue;
    const int st = ach % NST;
    mbar_wait(&full[st], (ach / NST) & 1);
    ++ach;
    const double2* A = ring + st * KC * R;
    // all operands of the chunk's KC/4 k-steps loaded before the first DMMA (their shared-memory
    // latencies overlap)
    double b[KC / 4][NT];
    double2 a[KC / 4][RT];
#pragma unroll
    for (int h = 0; h < KC / 4; ++h) {
      const int k0 = ch * KC + 4 * h;
#pragma unroll
      for (int t = 0; t < NT; ++t) b[h][t] = xd[(k0 + ac) * (2 * NS) + t * 8 + ar];
#pragma unroll
      for (int r = 0; r < RT; ++r) a[h][r] = A[(4 * h + ac) * R + (warp + r * NCW) * 8 + ar];
    }
#pragma unroll
    for (int h = 0; h < KC / 4; ++h)
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          dmma(c1[r][t][0], c1[r][t][1], a[h][r].x, b[h][t]);
          dmma(c2[r][t][0], c2[r][t][1], a[h][r].y, b[h][t]);
        }
    // the ring slot is refilled by the TMA (async proxy) after this release: order this warp's
    // generic-proxy reads of it first (without the fence a refill could overtake them; seen as
    // corrupted rows on nz = 64, 1 RHS)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int pk = (warp + r * NCW) * 8 + ar, pp = pk / nz, k = pk % nz;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int sl = t * 4 + ac;  // real columns 2 sl, 2 sl + 1
      const int item = sl % NI, cc = sl / NI, cx = cc & 1, cy = cc >> 1;
      if (item < p.n_items && cx < nkx && cy < nky) {
        double2 v = make_double2(c1[r][t][0] - c2[r][t][1], c1[r][t][1] + c2[r][t][0]);
        if ((pp == 0 && cx == 1) || (pp == 1 && cy == 1)) v = make_double2(-v.x, -v.y);
        p.X2[(long long)item * 3 * cs + pp * cs + k * zs + (long long)kys[cy] * Lx + kxs[cx]] = v;
      }
    }
  }
  pdl_trigger_late();
}

template <int NI, int RT>
static cudaError_t go_zlayer_tma(const ApplyParams& p, cudaStream_t s) {
  const int R = 3 * p.nz;
  constexpr int NST = NI == 1 ? 3 : 2;  // as in the kernel
  const size_t smem = (size_t)(R * 4 * NI + NST * 8 * R) * sizeof(double2) + 2 * NST * sizeof(uint64_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_zlayer_tma<NI, RT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  launch_pass(use_pdl(), k_zlayer_tma<NI, RT>, dim3((p.nx + 1) * (p.ny + 1)), dim3(288), smem, s, p);
  return cudaGetLastError();
}

template <int NI>
static cudaError_t go_zlayer_tma_r(const ApplyParams& p, cudaStream_t s) {
  // row tiles per consumer warp: R / 8 tiles over 8 warps
  const int tiles = 3 * p.nz / 8;
  switch (tiles) {
    case 24: return go_zlayer_tma<NI, 3>(p, s);  // nz = 64
    case 48: return go_zlayer_tma<NI, 6>(p, s);  // nz = 128
  }
  return cudaErrorInvalidValue;
}

template <int NI>
static cudaError_t go_zlayer_mma(const ApplyParams& p, cudaStream_t s) {
  constexpr int NSP = ((4 * NI + 7) / 8) * 8;
  const size_t smem = (size_t)3 * p.nz * NSP * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_zlayer_mma<NI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  launch_pass(use_pdl(), k_zlayer_mma<NI>, dim3((p.nx + 1) * (p.ny + 1)), dim3(256), smem, s, p);
  return cudaGetLastError();
}

template <int NI>
static cudaError_t go_zlayer(const ApplyParams& p, cudaStream_t s) {
  const size_t smem = (size_t)3 * p.nz * 4 * NI * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_zlayer<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e) return e;
  }
  const int R = 3 * p.nz;
  const int threads = std::min(256, ((R + 31) / 32) * 32);
  launch_pass(use_pdl(), k_zlayer<NI>, dim3((p.nx + 1) * (p.ny + 1)), dim3(threads), smem, s, p);
  return cudaGetLastError();
}

// IE_ZLAYER_MODE (side-by-side measurement): 0 (default) TMA ring + DMMA, 1 DMMA with direct
// loads, 2 DFMA
static int zlayer_mode() {
  static const int v = [] {
    const char* e = getenv("IE_ZLAYER_MODE");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// items of one launch share M (same domain); up to 3 (DMMA) or 4 (DFMA) per CTA, more by
// repeated launches
cudaError_t launch_zlayer(const ApplyParams& p, cudaStream_t s) {
  ApplyParams q = p;
  // the TMA-ring kernel is instantiated for 3nz/8 = 24 or 48 row tiles (nz = 64 or 128) only;
  // every other depth takes the direct-load DMMA or the DFMA kernel
  const bool tma = (p.nz == 64 || p.nz == 128) && zlayer_mode() == 0;
  const int group = tma ? 3 : 4;  // the DMMA kernel is best at <= 3
  for (int i0 = 0; i0 < p.n_items; i0 += group) {
    const int ni = std::min(group, p.n_items - i0);
    q.n_items = ni;
    for (int i = 0; i < ni; ++i) q.items[i] = p.items[i0 + i];
    const long long per_item = 3LL * p.nz * (2LL * p.ny) * (2LL * p.nx);
    q.X2 = p.X2 + (long long)i0 * per_item;
    cudaError_t e;
    const int mode = zlayer_mode();
    if (tma)  // DMMA fed by the TMA ring (3nz/8 row tiles over 8 warps)
      e = ni == 1 ? go_zlayer_tma_r<1>(q, s) : ni == 2 ? go_zlayer_tma_r<2>(q, s)
                  : ni == 3 ? go_zlayer_tma_r<3>(q, s) : go_zlayer_tma_r<4>(q, s);
    else if (ni >= 2 && p.nz % 8 == 0 && mode <= 1)  // DMMA, operands straight from global
      e = ni == 2 ? go_zlayer_mma<2>(q, s) : ni == 3 ? go_zlayer_mma<3>(q, s) : go_zlayer_mma<4>(q, s);
    else
      e = ni == 1 ? go_zlayer<1>(q, s) : ni == 2 ? go_zlayer<2>(q, s) : ni == 3 ? go_zlayer<3>(q, s) : go_zlayer<4>(q, s);
    if (e) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ receivers (table form)
// out[s][r] = h0[s][r] + (i omega mu0)^-1 sum_c E0rx_r(c) . (dsigma_c E_s(c)) dv: block partial
// sums in a fixed order, summed on the host in a fixed order.
__global__ void k_rx_table(const double2* __restrict__ E, const double2* __restrict__ E0rx,
                           const double* __restrict__ ds, long long N, int n_rx, double2* __restrict__ part) {
  const int pair = blockIdx.y, s = pair / n_rx, r = pair % n_rx;
  const double2* e = E + (long long)s * 3 * N;
  const double2* f = E0rx + (long long)r * 3 * N;
  double2 acc = czero();
  for (long long cidx = blockIdx.x * (long long)blockDim.x + threadIdx.x; cidx < N;
       cidx += (long long)gridDim.x * blockDim.x) {
    const double sxx = ds[cidx], syy = ds[N + cidx], szz = ds[2 * N + cidx];
    const double sxy = ds[3 * N + cidx], sxz = ds[4 * N + cidx], syz = ds[5 * N + cidx];
    const double2 e0 = e[cidx], e1 = e[N + cidx], e2 = e[2 * N + cidx];
    const double2 j0 = make_double2(sxx * e0.x + sxy * e1.x + sxz * e2.x, sxx * e0.y + sxy * e1.y + sxz * e2.y);
    const double2 j1 = make_double2(sxy * e0.x + syy * e1.x + syz * e2.x, sxy * e0.y + syy * e1.y + syz * e2.y);
    const double2 j2 = make_double2(sxz * e0.x + syz * e1.x + szz * e2.x, sxz * e0.y + syz * e1.y + szz * e2.y);
    acc = cadd(acc, cmul(f[cidx], j0));
    acc = cadd(acc, cmul(f[N + cidx], j1));
    acc = cadd(acc, cmul(f[2 * N + cidx], j2));
  }
  __shared__ double2 red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(long long)pair * gridDim.x + blockIdx.x] = red[0];
}

ie_status receivers_table(ie_ctx* c, const double2* e, int n_rx, const double2* e0rx, const cplx* h0, cplx* out,
                          double2* scratch, size_t scratch_elems) {
  const long long N = (long long)c->g.nx * c->g.ny * c->g.nz;
  const int pairs = c->n_src * n_rx;
  const int nblk = (int)std::max<long long>(1, std::min<long long>(256, (long long)scratch_elems / pairs));
  k_rx_table<<<dim3(nblk, pairs), 256, 0, c->stream>>>(e, e0rx, c->dsig, N, n_rx, scratch);
  IE_CHECK_LAUNCH(c, "k_rx_table");
  std::vector<double2> h((size_t)pairs * nblk);
  IE_CUDA(c, cudaMemcpyAsync(h.data(), scratch, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  IE_CUDA(c, cudaStreamSynchronize(c->stream));
  const double dv = c->g.dx * c->g.dy * c->g.dz;
  const cplx inv = 1.0 / cplx(0.0, c->omega * kMu0);
  for (int pr = 0; pr < pairs; ++pr) {
    cplx s = 0.0;
    for (int b = 0; b < nblk; ++b) s += cplx(h[(size_t)pr * nblk + b].x, h[(size_t)pr * nblk + b].y);
    out[pr] = h0[pr] + inv * s * dv;
  }
  return IE_OK;
}

}  // namespace ie
