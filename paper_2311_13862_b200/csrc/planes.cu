// Full-node ("FN") layout kernels for assembled problems with free boundary nodes
// (the reference's example-2: zero-flux face x = 1, problems.py:135-152) and the
// z-plane block smoothers of multigrid.py:48-110.
//
// Layout: one instance = all (c+1)^3 grid nodes of its level, x fastest, Dirichlet nodes
// held at zero.  Per instance and level the operator is a full-node 27-point coefficient
// array coefA[27][(c+1)^3] (row X, offset o: A[X, X+o]; zero rows on Dirichlet nodes and
// zero columns into them), combined from the batch-shared per-term arrays.  Every z-plane
// (c+1)^2 nodes) is contiguous, so the plane blocks of all instances are independent
// banded SPD systems of bandwidth c+2 (Dirichlet rows replaced by identity rows), factored
// once per parameter (banded Cholesky, one CTA per system) and solved with one warp per
// system.  The coarsest level is the same machinery with one 3D band system per instance.
#include "../../include/rbws_b200.h"
#include "common.cuh"

#include <cuda_runtime.h>
#include <cstdlib>
#include <type_traits>

namespace rbws {
namespace {

// band row stride: w+1 entries padded to whole 32-byte sectors
__host__ __device__ __forceinline__ int band_ws(int w) { return (w + 1 + 3) & ~3; }

__device__ __forceinline__ void o27_split(int o, int& dx, int& dy, int& dz) {
  dx = o % 3 - 1;
  dy = (o / 3) % 3 - 1;
  dz = o / 9 - 1;
}

// coefA[i][o][X] = sum_q theta[i][q] coef[q][o][X], terms in order, separately rounded
// (the reference's sum of scaled CSR terms, grid.py:246-255)
__global__ void fn_combine_kernel(int count, int Q, int64_t nodes, const double* __restrict__ theta,
                                  const double* __restrict__ coef, double* __restrict__ out) {
  const int64_t per = 27 * nodes;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (t >= per || i >= count) return;
  double acc = __dmul_rn(theta[i * Q], coef[t]);
  for (int q = 1; q < Q; ++q) acc = __dadd_rn(acc, __dmul_rn(theta[i * Q + q], coef[q * per + t]));
  out[i * per + t] = acc;
}

// mode 0: y = A x; mode 1: y = b - A x.  Row sums in ascending column order (CSR matvec)
__global__ void fn_apply_kernel(int count, int c, const double* __restrict__ coefA,
                                const double* __restrict__ x, const double* __restrict__ b,
                                double* __restrict__ y, int mode) {
  const int c1 = c + 1;
  const int64_t nodes = (int64_t)c1 * c1 * c1;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (X >= nodes) return;
  const int ix = (int)(X % c1), iy = (int)((X / c1) % c1), iz = (int)(X / ((int64_t)c1 * c1));
  const double* ca = coefA + (int64_t)i * 27 * nodes + X;
  const double* xi = x + (int64_t)i * nodes;
  double s = 0.0;
#pragma unroll
  for (int o = 0; o < 27; ++o) {
    int dx, dy, dz;
    o27_split(o, dx, dy, dz);
    const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
    if (jx < 0 || jx > c || jy < 0 || jy > c || jz < 0 || jz > c) continue;
    const double a = ca[o * nodes];
    if (a != 0.0) s = __dadd_rn(s, __dmul_rn(a, xi[X + dx + (int64_t)c1 * (dy + (int64_t)c1 * dz)]));
  }
  const int64_t g = (int64_t)i * nodes + X;
  y[g] = mode == 0 ? s : __dsub_rn(b[g], s);
}

// The same apply from the batch-shared per-term coefficients (no per-instance copy):
// each thread serves node X for IPT instances, combining theta_q coef_q[o][X] on the fly
// in the combine kernel's order and rounding, so the result is bitwise fn_apply_kernel's.
// Instance groups are the fastest grid dimension: the CTAs resident together work on the
// same nodes and the term coefficients come from L2.
template <int IPT>
__global__ void __launch_bounds__(256) fn_apply_shared_kernel(int count, int Q, int c,
                                                              const double* __restrict__ theta,
                                                              const double* __restrict__ coef,
                                                              const double* __restrict__ x,
                                                              const double* __restrict__ b,
                                                              double* __restrict__ y, int mode) {
  const int c1 = c + 1;
  const int64_t nodes = (int64_t)c1 * c1 * c1;
  const int groups = (count + IPT - 1) / IPT;
  const int grp = blockIdx.x % groups;
  const int64_t X = (int64_t)(blockIdx.x / groups) * blockDim.x + threadIdx.x;
  if (X >= nodes) return;
  const int i0 = grp * IPT;
  const int ix = (int)(X % c1), iy = (int)((X / c1) % c1), iz = (int)(X / ((int64_t)c1 * c1));
  double th[IPT][kMaxTerms];
#pragma unroll
  for (int u = 0; u < IPT; ++u)
#pragma unroll
    for (int q = 0; q < kMaxTerms; ++q)
      th[u][q] = (q < Q && i0 + u < count) ? theta[(i0 + u) * Q + q] : 0.0;
  double sacc[IPT];
#pragma unroll
  for (int u = 0; u < IPT; ++u) sacc[u] = 0.0;
  const int64_t per = 27 * nodes;
#pragma unroll 3
  for (int o = 0; o < 27; ++o) {
    int dx, dy, dz;
    o27_split(o, dx, dy, dz);
    const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
    if (jx < 0 || jx > c || jy < 0 || jy > c || jz < 0 || jz > c) continue;
    const int64_t off = X + dx + (int64_t)c1 * (dy + (int64_t)c1 * dz);
    double cq[kMaxTerms];
#pragma unroll
    for (int q = 0; q < kMaxTerms; ++q) cq[q] = q < Q ? coef[q * per + o * nodes + X] : 0.0;
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      if (i0 + u >= count) break;
      double a = __dmul_rn(th[u][0], cq[0]);
#pragma unroll
      for (int q = 1; q < kMaxTerms; ++q)
        if (q < Q) a = __dadd_rn(a, __dmul_rn(th[u][q], cq[q]));
      if (a != 0.0)
        sacc[u] = __dadd_rn(sacc[u], __dmul_rn(a, x[(int64_t)(i0 + u) * nodes + off]));
    }
  }
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    if (i0 + u >= count) break;
    const int64_t g = (int64_t)(i0 + u) * nodes + X;
    y[g] = mode == 0 ? sacc[u] : __dsub_rn(b[g], sacc[u]);
  }
}

// block Gauss-Seidel right-hand side of z-plane p (multigrid.py:79-89):
// out[i][r] = (b - A[p, p-1] x_{p-1}) - A[p, p+1] x_{p+1} at node r of the plane
__global__ void fn_plane_rhs_kernel(int count, int c, int p, const double* __restrict__ coefA,
                                    const double* __restrict__ x, const double* __restrict__ b,
                                    double* __restrict__ out) {
  const int c1 = c + 1;
  const int64_t nodes = (int64_t)c1 * c1 * c1, M = (int64_t)c1 * c1;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (r >= M) return;
  const int64_t X = p * M + r;
  const int ix = (int)(r % c1), iy = (int)(r / c1);
  const double* ca = coefA + (int64_t)i * 27 * nodes + X;
  const double* xi = x + (int64_t)i * nodes;
  double sp = 0.0, sn = 0.0;
#pragma unroll
  for (int o = 0; o < 27; ++o) {
    int dx, dy, dz;
    o27_split(o, dx, dy, dz);
    if (dz == 0) continue;
    const int jx = ix + dx, jy = iy + dy, jz = p + dz;
    if (jx < 0 || jx > c || jy < 0 || jy > c || jz < 0 || jz > c) continue;
    const double a = ca[o * nodes];
    if (a == 0.0) continue;
    const double t = __dmul_rn(a, xi[X + dx + (int64_t)c1 * (dy + (int64_t)c1 * dz)]);
    if (dz < 0) sp = __dadd_rn(sp, t);
    else sn = __dadd_rn(sn, t);
  }
  out[(int64_t)i * M + r] = __dsub_rn(__dsub_rn(b[(int64_t)i * nodes + X], sp), sn);
}

// lower band of the plane blocks (planar = 1: systems = instances x planes, M = (c+1)^2,
// w = c+2) or of the whole level (planar = 0: M = (c+1)^3, w = (c+1)^2 + c + 2):
// band[(s*M + r)*ws + d] = A[r, r-d] (ws = band_ws(w)); Dirichlet rows -> identity rows
__global__ void fn_band_build_kernel(int count, int c, int planar, const double* __restrict__ coefA,
                                     double* __restrict__ band) {
  const int c1 = c + 1;
  const int64_t nodes = (int64_t)c1 * c1 * c1;
  const int64_t M = planar ? (int64_t)c1 * c1 : nodes;
  const int w = planar ? c + 2 : c1 * c1 + c + 2;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (X >= nodes) return;
  const int ix = (int)(X % c1), iy = (int)((X / c1) % c1), iz = (int)(X / ((int64_t)c1 * c1));
  const int64_t s = planar ? (int64_t)i * c1 + iz : i;
  const int64_t r = planar ? X - (int64_t)iz * c1 * c1 : X;
  const int ws = band_ws(w);
  double* row = band + (s * M + r) * ws;
  for (int d = 0; d < ws; ++d) row[d] = 0.0;
  const double* ca = coefA + (int64_t)i * 27 * nodes + X;
  const double dg = ca[13 * nodes];
  if (dg == 0.0) {  // Dirichlet node: decoupled identity row
    row[0] = 1.0;
    return;
  }
  for (int o = 0; o <= 13; ++o) {
    int dx, dy, dz;
    o27_split(o, dx, dy, dz);
    if (planar && dz != 0) continue;
    const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
    if (jx < 0 || jx > c || jy < 0 || jy > c || jz < 0 || jz > c) continue;
    const int d = -(dx + c1 * (dy + c1 * dz));
    row[d] = ca[o * nodes];
  }
}

// banded Cholesky in place, one CTA per system (right-looking, column j's trailing
// (w x w) triangle updated in parallel); the diagonal slot of row j ends as 1 / L_jj;
// info[s] = 0 or the first non-positive pivot + 1
__global__ void band_factor_kernel(int64_t nsys, int64_t M, int w, double* __restrict__ band,
                                   int* __restrict__ info) {
  const int64_t s = blockIdx.x;
  if (s >= nsys) return;
  const int ws = band_ws(w);
  double* B = band + s * M * ws;
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t j = 0; j < M; ++j) {
    if (threadIdx.x == 0) {
      const double a = B[j * ws];
      if (!(a > 0.0) && !bad) bad = (int)(j + 1);
      piv = a > 0.0 ? sqrt(a) : 1.0;
      B[j * ws] = piv;
    }
    __syncthreads();
    const double p = piv;
    for (int t = 1 + threadIdx.x; t <= w; t += blockDim.x)
      if (j + t < M) B[(j + t) * ws + t] /= p;
    // the diagonal slot keeps 1 / L_jj: the solves multiply (no division on their chains)
    if (threadIdx.x == 0) B[j * ws] = 1.0 / p;
    __syncthreads();
    // A[j+a][j+b] -= L[j+a][j] L[j+b][j], 1 <= b <= a <= w
    for (int a = 1 + warp; a <= w; a += nw) {
      if (j + a >= M) break;
      const double la = B[(j + a) * ws + a];
      for (int bb = 1 + lane; bb <= a; bb += 32)
        B[(j + a) * ws + (a - bb)] -= la * B[(j + bb) * ws + bb];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) info[s] = bad;
}

// The same factorization with the active (w+1)-row window in shared memory (row r in
// slot r mod (w+1)): the per-step read-modify-write of the trailing triangle stays on
// chip (in global memory every step wrote ~w^2/2 doubles through to L2); row j leaves
// for HBM when final, row j+w+1 enters from the assembled band just before its first
// update.
constexpr int kFacK = 5;  // shared-window factorization: bandwidths w < 32 kFacK

__global__ void __launch_bounds__(256) band_factor_smem_kernel(int64_t nsys, int64_t M, int w,
                                                               double* __restrict__ band,
                                                               int* __restrict__ info) {
  extern __shared__ double wnd[];
  const int64_t s = blockIdx.x;
  if (s >= nsys) return;
  const int ws = band_ws(w), W1 = w + 1, NS = w + 2;  // one spare slot: see below
  double* B = band + s * M * ws;
  __shared__ int bad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) bad = 0;
  for (int t = threadIdx.x; t < W1 * ws; t += blockDim.x) {
    const int row = t / ws;
    wnd[t] = row < M ? B[(int64_t)row * ws + t % ws] : 0.0;
  }
  __syncthreads();
  // rows j..j+w live in slots jm.. (mod w+2); the spare slot (that of row j-1, already
  // written out) receives row j+w+1 while step j updates, so a step needs two barriers
  int jm = 0;
  auto rowp = [&](int x) {  // row j + x, 0 <= x <= w+1
    const int t = jm + x;
    return wnd + (t >= NS ? t - NS : t) * ws;
  };
  for (int64_t j = 0; j < M; ++j) {
    double* rj = rowp(0);
    const double a0 = rj[0];  // every thread derives the pivot itself (no broadcast barrier)
    const double p = a0 > 0.0 ? sqrt(a0) : 1.0;
    if (threadIdx.x == 0 && !(a0 > 0.0) && !bad) bad = (int)(j + 1);
    for (int t = 1 + threadIdx.x; t <= w; t += blockDim.x)
      if (j + t < M) rowp(t)[t] /= p;
    __syncthreads();
    // column j (L[j+bb][j], bb = lane + 1 + 32k) in registers: the same for every row
    double colv[kFacK];
#pragma unroll
    for (int k = 0; k < kFacK; ++k) {
      const int bb = lane + 1 + 32 * k;
      colv[k] = (bb <= w && j + bb < M) ? rowp(bb)[bb] : 0.0;
    }
    for (int a = 1 + warp; a <= w; a += nw) {
      if (j + a >= M) break;
      double* ra = rowp(a);
      const double la = ra[a];
#pragma unroll
      for (int k = 0; k < kFacK; ++k) {
        const int bb = lane + 1 + 32 * k;
        if (bb <= a) ra[a - bb] -= la * colv[k];
      }
    }
    // row j is final: out to HBM (diagonal slot = 1 / L_jj); row j+w+1 into the spare slot
    for (int t = threadIdx.x; t < ws; t += blockDim.x) B[j * ws + t] = t == 0 ? 1.0 / p : rj[t];
    if (j + W1 < M) {
      double* rn = rowp(W1);
      for (int t = threadIdx.x; t < ws; t += blockDim.x) rn[t] = B[(j + W1) * ws + t];
    }
    jm = (jm + 1 == NS) ? 0 : jm + 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) info[s] = bad;
}

// Blocked (panel) variant: NB columns per step.  The window holds rows j .. j+w+NB-1 (row r
// in slot r mod (w+NB)).  Per panel: (1) the NB x NB diagonal block is factored by one warp
// (lane r = row j+r, columns broadcast by shuffles), (2) the w trailing rows' panel entries
// are solved against it (one thread per row, L_D entries broadcast from shared memory),
// (3) the trailing w x w triangle takes the rank-NB update as 4 x 4 register tiles (SYRK),
// (4) the panel rows leave for HBM (diagonal slot = 1 / L_jj) and the next NB band rows
// enter.  Four barriers per NB rows instead of two per row; the same arithmetic as the
// right-looking kernels up to the order of the trailing sums.
#ifndef RBWS_BF_TPB
#define RBWS_BF_TPB 128
#endif
template <int NB>
__global__ void __launch_bounds__(RBWS_BF_TPB, 4) band_factor_blk_kernel(int64_t nsys, int64_t M, int w,
                                                             double* __restrict__ band,
                                                             int* __restrict__ info) {
  extern __shared__ double wnd[];
  const int64_t s = blockIdx.x;
  if (s >= nsys) return;
  const int ws = band_ws(w), R = w + NB;
  double* B = band + s * M * ws;
  __shared__ int bad;
  __shared__ double dinvp[NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad = 0;
  auto row = [&](int64_t r) -> double* { return wnd + (int)(r % R) * ws; };
  for (int t = tid; t < R * ws; t += blockDim.x) {
    const int r = t / ws;
    wnd[t] = r < M ? B[(int64_t)r * ws + t % ws] : 0.0;
  }
  __syncthreads();
  const int TA = (w + 3) / 4, ntiles = TA * (TA + 1) / 2;
  for (int64_t j = 0; j < M; j += NB) {
    const int nbe = (int)(M - j < NB ? M - j : NB);
    // (1) diagonal block
    if (warp == 0) {
      double a[NB];
      double* rr = row(j + (lane < nbe ? lane : 0));
#pragma unroll
      for (int c = 0; c < NB; ++c) a[c] = (lane < nbe && c <= lane && lane - c <= w) ? rr[lane - c] : 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c < nbe) {
          const double pv = __shfl_sync(0xffffffffu, a[c], c);
          const bool ok = pv > 0.0;
          if (lane == 0 && !ok && !bad) bad = (int)(j + c + 1);
          // 1/sqrt by the hardware estimate + two Newton steps (no DSQRT / DDIV sequence on
          // the panel's critical path), L = pv / sqrt(pv)
          const double q = ok ? pv : 1.0;
          double inv = rsqrt(q);
          inv = inv * fma(-0.5 * q, inv * inv, 1.5);
          inv = inv * fma(-0.5 * q, inv * inv, 1.5);
          const double L = q * inv;
          if (lane == c) {
            a[c] = L;
            dinvp[c] = inv;
          } else if (lane > c) {
            a[c] *= inv;
          }
#pragma unroll
          for (int c2 = c + 1; c2 < NB; ++c2) {
            const double l2 = __shfl_sync(0xffffffffu, a[c], c2);
            if (lane >= c2 && c2 < nbe) a[c2] = fma(-a[c], l2, a[c2]);
          }
        }
      }
      if (lane < nbe) {
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c <= lane && lane - c <= w) rr[lane - c] = a[c];
      }
    }
    __syncthreads();
    // (2) panel entries of the trailing rows
    const int64_t t0 = j + nbe;
    for (int tr = tid; tr < w && t0 + tr < M; tr += blockDim.x) {
      const int64_t rr = t0 + tr;
      double* rw = row(rr);
      double x[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int64_t d = rr - j - c;
        x[c] = (c < nbe && d <= w) ? rw[d] : 0.0;
      }
      // column-oriented: x_c is final after its scaling, then eliminated from the later
      // columns (16 short steps instead of one 120-FMA dependent chain)
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c < nbe) {
          x[c] *= dinvp[c];
#pragma unroll
          for (int c2 = c + 1; c2 < NB; ++c2)
            if (c2 < nbe && c2 - c <= w) x[c2] = fma(-x[c], row(j + c2)[c2 - c], x[c2]);
        }
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int64_t d = rr - j - c;
        if (c < nbe && d <= w) rw[d] = x[c];
      }
    }
    __syncthreads();
    // (3) trailing update A[t0+a][t0+b] -= sum_c L[t0+a][j+c] L[t0+b][j+c], b <= a < w
    for (int tt = tid; tt < ntiles; tt += blockDim.x) {
      int ta = 0;
      while ((ta + 1) * (ta + 2) / 2 <= tt) ++ta;
      const int tb = tt - ta * (ta + 1) / 2;
      double acc[4][4];
      const double* ra[4];
      const double* cb[4];
      int64_t da[4], db[4];
      bool oka[4], okb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = t0 + ta * 4 + u, cc = t0 + tb * 4 + u;
        oka[u] = ta * 4 + u < w && rr < M;
        okb[u] = tb * 4 + u < w && cc < M;
        ra[u] = row(oka[u] ? rr : t0);
        cb[u] = row(okb[u] ? cc : t0);
        da[u] = rr - j;
        db[u] = cc - j;
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      }
      for (int c = 0; c < nbe; ++c) {
        double pa[4], pb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          pa[u] = (oka[u] && da[u] - c <= w) ? ra[u][da[u] - c] : 0.0;
          pb[u] = (okb[u] && db[u] - c <= w) ? cb[u][db[u] - c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(pa[u], pb[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int a = ta * 4 + u;
        const int64_t rr = t0 + a;
        if (a >= w || rr >= M) continue;
        double* rw = row(rr);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int b = tb * 4 + v;
          if (b <= a) rw[a - b] -= acc[u][v];
        }
      }
    }
    __syncthreads();
    // (4) panel rows out (diagonal slot 1 / L_jj), next band rows in
    for (int t = tid; t < nbe * ws; t += blockDim.x) {
      const int c = t / ws, d = t % ws;
      B[(j + c) * ws + d] = d == 0 ? dinvp[c] : row(j + c)[d];
    }
    __syncthreads();
    for (int t = tid; t < nbe * ws; t += blockDim.x) {
      const int64_t r = j + R + t / ws;
      row(r)[t % ws] = r < M ? B[r * ws + t % ws] : 0.0;
    }
    __syncthreads();
  }
  if (tid == 0) info[s] = bad;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// L L^T z = r per system (one warp each): forward into r, backward into a shared ring;
// mode 0: x = z; mode 1: x += omega z (damped plane-Jacobi update)
__global__ void band_solve_kernel(int64_t nsys, int64_t M, int w, int ring,
                                  const double* __restrict__ L, double* __restrict__ r,
                                  double* __restrict__ x, double omega, int mode) {
  extern __shared__ double sring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (s >= nsys) return;
  double* zr = sring + warp * ring;
  const int rm = ring - 1;
  const int ws = band_ws(w);
  const double* Ls = L + s * M * ws;
  double* rs = r + s * M;
  double* xs = x + s * M;
  for (int64_t i = 0; i < M; ++i) {
    const double* li = Ls + i * ws;
    double acc = 0.0;
    for (int d = 1 + lane; d <= w; d += 32)
      if (i - d >= 0) acc += li[d] * zr[(i - d) & rm];
    acc = warp_sum(acc);
    const double y = (rs[i] - acc) * li[0];
    __syncwarp();
    if (lane == 0) {
      zr[i & rm] = y;
      rs[i] = y;
    }
    __syncwarp();
  }
  for (int64_t i = M - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int d = 1 + lane; d <= w; d += 32)
      if (i + d < M) acc += Ls[(i + d) * ws + d] * zr[(i + d) & rm];
    acc = warp_sum(acc);
    const double z = (rs[i] - acc) * Ls[i * ws];
    __syncwarp();
    if (lane == 0) {
      zr[i & rm] = z;
      xs[i] = mode == 0 ? z : xs[i] + omega * z;
    }
    __syncwarp();
  }
}

// Sub-warp variant: LPS lanes per system (32/LPS systems per warp); lane j of a system
// holds band entries d = j + LPS k (k < KPS) of a row.  The M-step chains are latency
// bound and the row work is tiny (w FMAs), so nothing on the chain touches memory: the
// window of the last w solution values lives in registers (slot d of the window on the
// lane owning d) and moves one slot per step by shuffles, and the rows of the next PF
// steps are loaded into registers ahead of the chain.  (A shared-memory window needs a
// __syncwarp per step, whose memory-ordering semantics make every step wait for the
// prefetch loads in flight: measured 1.4-1.9 us per step.)
// Forward: row form, y_i = (r_i - sum_d L[i][i-d] y_{i-d}) / L_ii (log2(LPS)-level
// reduction).  Backward: column form on ROWS of L (no strided column reads, no
// reduction): z_i = p_0 / L_ii, p_d -= L[i][i-d] z_i, then the window shifts and entry
// i-1-w enters it with its forward value.
template <int LPS, int KPS, int PF>
__global__ void __launch_bounds__(128) band_solve_sub_kernel(int64_t nsys, int64_t M, int w,
                                                             const double* __restrict__ L,
                                                             int64_t lstride,
                                                             double* __restrict__ r, int64_t rstride,
                                                             double* __restrict__ x, int64_t xstride,
                                                             double omega, int mode) {
  constexpr int SPW = 32 / LPS;  // systems per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPS, j = lane % LPS;
  const int64_t s = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * SPW + g;
  if (s >= nsys) return;  // whole groups only (a group = one system)
  const unsigned gmask = (LPS == 32) ? 0xffffffffu : (((1u << LPS) - 1u) << (g * LPS));
  const int W1 = band_ws(w);
  const int jw = w % LPS, kw = w / LPS;  // owner of d = w
  const double* Ls = L + s * lstride;  // system strides (contiguous: M W1, M, M)
  double* rs = r + s * rstride;
  double* xs = x + s * xstride;
  double buf[PF][KPS], ga[PF], gb[PF];
  double win[KPS];
#pragma unroll
  for (int k = 0; k < KPS; ++k) win[k] = 0.0;
  auto load_row = [&](int64_t i, int u, bool fwd) {
    const bool ok = i >= 0 && i < M;
#pragma unroll
    for (int k = 0; k < KPS; ++k) {
      const int d = j + LPS * k;
      buf[u][k] = (ok && d <= w) ? __ldcs(Ls + i * W1 + d) : 0.0;
    }
    if (fwd) {
      ga[u] = (ok && j == 0) ? rs[i] : 0.0;
    } else {  // y_{i-1-w}: enters the window after step i
      ga[u] = (ok && j == jw && i - 1 - w >= 0) ? rs[i - 1 - w] : 0.0;
      gb[u] = (ok && j == 0 && mode == 1) ? xs[i] : 0.0;
    }
  };
  // ---- forward: L y = r; window slot d holds y_{i-d} (d >= 1)
#pragma unroll
  for (int u = 0; u < PF; ++u) load_row(u, u, true);
  for (int64_t i0 = 0; i0 < M; i0 += PF) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int64_t i = i0 + u;
      if (i < M) {
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int k = 0; k < KPS; ++k) {
          if (k & 1) acc1 = fma(buf[u][k], win[k], acc1);  // slot 0 and slots past w hold 0
          else acc0 = fma(j == 0 && k == 0 ? 0.0 : buf[u][k], win[k], acc0);
        }
        double acc = acc0 + acc1;
#pragma unroll
        for (int o = LPS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o, LPS);
        const double y = (__shfl_sync(gmask, ga[u], 0, LPS) - acc) * __shfl_sync(gmask, buf[u][0], 0, LPS);
        if (j == 0) rs[i] = y;
        // shift: slot d+1 <- slot d, slot 1 <- y_i; slots past w drop out (zeroed)
        double nw[KPS];
#pragma unroll
        for (int k = 0; k < KPS; ++k) {
          const double up = __shfl_up_sync(gmask, win[k], 1, LPS);
          const double wrap = __shfl_sync(gmask, k > 0 ? win[k - 1] : y, LPS - 1, LPS);
          nw[k] = (j == 0) ? (k == 0 ? 0.0 : wrap) : up;
        }
        // lane 1 (or lane 0's next slot when LPS == 1) receives y_i into slot 1
#pragma unroll
        for (int k = 0; k < KPS; ++k) {
          const int d = j + LPS * k;
          win[k] = (d == 1) ? y : (d > w ? 0.0 : nw[k]);
        }
      }
      load_row(i + PF, u, true);
    }
  }
  __syncwarp(gmask);  // the forward values in rs are read back by other lanes below
  // ---- backward: L^T z = y; window slot d holds the pending value of entry i-d
#pragma unroll
  for (int k = 0; k < KPS; ++k) {
    const int d = j + LPS * k;
    win[k] = (d <= w && M - 1 - d >= 0) ? rs[M - 1 - d] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PF; ++u) load_row(M - 1 - u, u, false);
  for (int64_t i0 = M - 1; i0 >= 0; i0 -= PF) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int64_t i = i0 - u;
      if (i >= 0) {
        const double z = __shfl_sync(gmask, win[0], 0, LPS) * __shfl_sync(gmask, buf[u][0], 0, LPS);
        if (j == 0) xs[i] = mode == 0 ? z : gb[u] + omega * z;
#pragma unroll
        for (int k = 0; k < KPS; ++k) win[k] = fma(-buf[u][k], z, win[k]);  // (slot 0 unused after)
        // shift: slot d <- slot d+1; slot w <- y_{i-1-w}
        double nw[KPS];
#pragma unroll
        for (int k = 0; k < KPS; ++k) {
          const double dn = __shfl_down_sync(gmask, win[k], 1, LPS);
          const double wrap = __shfl_sync(gmask, k + 1 < KPS ? win[k + 1] : 0.0, 0, LPS);
          nw[k] = (j == LPS - 1) ? wrap : dn;
        }
#pragma unroll
        for (int k = 0; k < KPS; ++k) win[k] = (j == jw && k == kw) ? ga[u] : nw[k];
      }
      load_row(i - PF, u, false);
    }
  }
}

// The band factor transposed: U[i][d] = L[i+d][i] (= band[(i+d) ws + d]), U[i][0] = 1 / L_ii.
// Row i of U is column i of L, i.e. what the forward substitution scatters once y_i is known.
__global__ void band_transpose_kernel(int64_t nsys, int64_t M, int w, const double* __restrict__ band,
                                      double* __restrict__ bandT) {
  const int ws = band_ws(w);
  const int64_t s = blockIdx.y;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (i, d) of the output
  if (s >= nsys || t >= M * ws) return;
  const int64_t i = t / ws;
  const int d = (int)(t % ws);
  const double* B = band + s * M * ws;
  bandT[s * M * ws + t] = (d <= w && i + d < M) ? B[(i + d) * ws + d] : 0.0;
}

// L L^T z = r per system with one warp and no reductions on the dependency chain.  Both
// substitutions run in scatter form: when y_i (forward, rows of U = L^T) or x_i (backward,
// rows of L) is final, the pending values of the w rows it couples to are updated at once.
// Rows are owned round-robin (row t by lane t mod 32, slot = 32-row group, SL slots cover the
// w + 32 rows in flight), so the next row's owner is the next lane and the chain per row is
// one multiply, one shuffle broadcast and one FMA (no shifting window, no dot-product
// reduction); the row loads are coalesced and independent of the chain.
// mode 0: x = z; mode 1: x += omega z.  r is overwritten with the forward result.
template <int SL>
__global__ void __launch_bounds__(128) band_solve_rot_kernel(int64_t nsys, int64_t M, int w,
                                                             const double* __restrict__ L,
                                                             const double* __restrict__ U,
                                                             int64_t lstride,
                                                             double* __restrict__ r, int64_t rstride,
                                                             double* __restrict__ x, int64_t xstride,
                                                             double omega, int mode) {
#ifndef RBWS_ROT_PF
#define RBWS_ROT_PF 8
#endif
  constexpr int PF = RBWS_ROT_PF;  // rows loaded ahead of the chain (registers: PF x SL)
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nsys) return;
  const int ws = band_ws(w);
  const double* Ls = L + s * lstride;
  const double* Us = U + s * lstride;
  double* rs = r + s * rstride;
  double* xs = x + s * xstride;
  const int64_t G = (M + 31) / 32;
  double p[SL];
  double buf[PF][SL];
  // row i's entries for this lane's slots: forward d = 32 m + lane - (i mod 32) of U row i,
  // backward d = 32 m + (i mod 32) - lane of L row i
  auto load_fwd = [&](int64_t i, double* b) {
    const int o = (int)(i & 31);
#pragma unroll
    for (int m = 0; m < SL; ++m) {
      const int d = 32 * m + lane - o;
      b[m] = (i < M && d >= 0 && d <= w) ? __ldcs(Us + i * ws + d) : 0.0;
    }
  };
  auto load_bwd = [&](int64_t i, double* b) {
    const int o = (int)(i & 31);
#pragma unroll
    for (int m = 0; m < SL; ++m) {
      const int d = 32 * m + o - lane;
      b[m] = (i >= 0 && i < M && d >= 0 && d <= w) ? __ldcs(Ls + i * ws + d) : 0.0;
    }
  };
  // ---- forward L y = r (scatter with the rows of U); slot m <-> row 32 (q + m) + lane
#pragma unroll
  for (int m = 0; m < SL; ++m) {
    const int64_t t = 32 * m + lane;
    p[m] = t < M ? rs[t] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PF; ++u) load_fwd(u, buf[u]);
  for (int64_t q = 0; q < G; ++q) {
#pragma unroll
    for (int o0 = 0; o0 < 32; o0 += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int o = o0 + u;
        const int64_t i = 32 * q + o;
        if (i < M) {
          const double z = __shfl_sync(0xffffffffu, p[0] * buf[u][0], o);  // lane o: row i
          if (lane == o) rs[i] = z;
#pragma unroll
          for (int m = 0; m < SL; ++m) {
            const int d = 32 * m + lane - o;
            if (d >= 1 && d <= w) p[m] = fma(-buf[u][m], z, p[m]);
          }
        }
        load_fwd(i + PF, buf[u]);
      }
    }
#pragma unroll
    for (int m = 0; m + 1 < SL; ++m) p[m] = p[m + 1];
    const int64_t t = 32 * (q + SL) + lane;
    p[SL - 1] = t < M ? rs[t] : 0.0;
  }
  __syncwarp();
  // ---- backward L^T x = y (scatter with the rows of L); slot m <-> row 32 (q - m) + lane
#pragma unroll
  for (int m = 0; m < SL; ++m) {
    const int64_t t = 32 * (G - 1 - m) + lane;
    p[m] = (t >= 0 && t < M) ? rs[t] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PF; ++u) load_bwd(32 * G - 1 - u, buf[u]);
  for (int64_t q = G - 1; q >= 0; --q) {
#pragma unroll
    for (int o0 = 31; o0 >= 0; o0 -= PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int o = o0 - u;
        const int64_t i = 32 * q + o;
        if (i < M) {
          const double z = __shfl_sync(0xffffffffu, p[0] * buf[u][0], o);
          if (lane == o) xs[i] = mode == 0 ? z : fma(omega, z, xs[i]);
#pragma unroll
          for (int m = 0; m < SL; ++m) {
            const int d = 32 * m + o - lane;
            if (d >= 1 && d <= w) p[m] = fma(-buf[u][m], z, p[m]);
          }
        }
        load_bwd(i - PF, buf[u]);
      }
    }
#pragma unroll
    for (int m = 0; m + 1 < SL; ++m) p[m] = p[m + 1];
    const int64_t t = 32 * (q - SL) + lane;
    p[SL - 1] = t >= 0 ? rs[t] : 0.0;
  }
}

// b[I] = sum_a w(a) r[2I + a] over the 27 fine neighbours (ascending fine index: the
// reference's P^T r), zero on coarse Dirichlet nodes (cmask)
__global__ void fn_restrict_kernel(int count, int cc, const double* __restrict__ r,
                                   double* __restrict__ b, const unsigned char* __restrict__ cmask) {
  const int c1 = cc + 1, f1 = 2 * cc + 1;
  const int64_t cn = (int64_t)c1 * c1 * c1, fn = (int64_t)f1 * f1 * f1;
  const int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (I >= cn) return;
  double s = 0.0;
  if (cmask[I]) {
    const int ix = (int)(I % c1), iy = (int)((I / c1) % c1), iz = (int)(I / ((int64_t)c1 * c1));
    const double* ri = r + (int64_t)i * fn;
    for (int az = -1; az <= 1; ++az) {
      const int fz = 2 * iz + az;
      if (fz < 0 || fz >= f1) continue;
      for (int ay = -1; ay <= 1; ++ay) {
        const int fy = 2 * iy + ay;
        if (fy < 0 || fy >= f1) continue;
        for (int ax = -1; ax <= 1; ++ax) {
          const int fx = 2 * ix + ax;
          if (fx < 0 || fx >= f1) continue;
          const double wgt = (ax ? 0.5 : 1.0) * (ay ? 0.5 : 1.0) * (az ? 0.5 : 1.0);
          s = __dadd_rn(s, __dmul_rn(wgt, ri[fx + (int64_t)f1 * (fy + (int64_t)f1 * fz)]));
        }
      }
    }
  }
  b[(int64_t)i * cn + I] = s;
}

// u[X] += (P e)[X] on fine free nodes (trilinear; coarse columns ascending)
__global__ void fn_prolong_kernel(int count, int cc, const double* __restrict__ e,
                                  double* __restrict__ u, const unsigned char* __restrict__ fmask) {
  const int c1 = cc + 1, f1 = 2 * cc + 1;
  const int64_t cn = (int64_t)c1 * c1 * c1, fn = (int64_t)f1 * f1 * f1;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (X >= fn || !fmask[X]) return;
  const int fx = (int)(X % f1), fy = (int)((X / f1) % f1), fz = (int)(X / ((int64_t)f1 * f1));
  const double* ei = e + (int64_t)i * cn;
  int lo[3], hi[3];
  const int f[3] = {fx, fy, fz};
  for (int a = 0; a < 3; ++a) {
    lo[a] = f[a] >> 1;
    hi[a] = (f[a] & 1) ? lo[a] + 1 : lo[a];
  }
  double s = 0.0;
  for (int kz = lo[2]; kz <= hi[2]; ++kz)
    for (int ky = lo[1]; ky <= hi[1]; ++ky)
      for (int kx = lo[0]; kx <= hi[0]; ++kx) {
        const double wgt = (lo[0] == hi[0] ? 1.0 : 0.5) * (lo[1] == hi[1] ? 1.0 : 0.5) *
                           (lo[2] == hi[2] ? 1.0 : 0.5);
        s = __dadd_rn(s, __dmul_rn(wgt, ei[kx + (int64_t)c1 * (ky + (int64_t)c1 * kz)]));
      }
  const int64_t g = (int64_t)i * fn + X;
  u[g] = __dadd_rn(u[g], s);
}

// damped point Jacobi from a residual: x += omega r / diag on free nodes (kernels.py:98-115)
__global__ void fn_point_jacobi_kernel(int count, int64_t nodes, const double* __restrict__ coefA,
                                       const double* __restrict__ r, double* __restrict__ x,
                                       double omega) {
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (X >= nodes) return;
  const double d = coefA[((int64_t)i * 27 + 13) * nodes + X];
  const int64_t g = (int64_t)i * nodes + X;
  if (d != 0.0) x[g] = __dadd_rn(x[g], __ddiv_rn(__dmul_rn(omega, r[g]), d));
}

inline dim3 grid_of(int64_t n, int count, int t = 256) {
  return dim3((unsigned)((n + t - 1) / t), (unsigned)count);
}

inline int band_w(int c, int planar) { return planar ? c + 2 : (c + 1) * (c + 1) + c + 2; }

}  // namespace
}  // namespace rbws

using namespace rbws;

static inline cudaStream_t St(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define FN_LAUNCHED()                                   \
  do {                                                  \
    count_launch();                                     \
    RBWS_CUDA_CHECK(cudaGetLastError());                \
  } while (0)

extern "C" {

int rbws_fn_combine(int count, int nterms, int c, const double* theta, const double* coef,
                    double* coefA, void* stream) {
  if (count <= 0 || nterms <= 0 || c < 1 || !theta || !coef || !coefA)
    return rbws_set_error("rbws_fn_combine: bad argument", __FILE__, __LINE__);
  const int64_t nodes = (int64_t)(c + 1) * (c + 1) * (c + 1);
  fn_combine_kernel<<<grid_of(27 * nodes, count), 256, 0, St(stream)>>>(count, nterms, nodes, theta,
                                                                         coef, coefA);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_apply(int count, int c, const double* coefA, const double* x, const double* b,
                  double* y, int mode, void* stream) {
  if (count <= 0 || c < 1 || !coefA || !x || !y || (mode == 1 && !b) || mode < 0 || mode > 1)
    return rbws_set_error("rbws_fn_apply: bad argument", __FILE__, __LINE__);
  const int64_t nodes = (int64_t)(c + 1) * (c + 1) * (c + 1);
  fn_apply_kernel<<<grid_of(nodes, count), 256, 0, St(stream)>>>(count, c, coefA, x, b, y, mode);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_apply_shared(int count, int nterms, int c, const double* theta, const double* coef,
                         const double* x, const double* b, double* y, int mode, void* stream) {
  if (count <= 0 || nterms <= 0 || nterms > kMaxTerms || c < 1 || !theta || !coef || !x || !y ||
      (mode == 1 && !b) || mode < 0 || mode > 1)
    return rbws_set_error("rbws_fn_apply_shared: bad argument", __FILE__, __LINE__);
  const int64_t nodes = (int64_t)(c + 1) * (c + 1) * (c + 1);
  constexpr int IPT = 4;
  const int64_t groups = (count + IPT - 1) / IPT;
  const int64_t blocks = ((nodes + 255) / 256) * groups;
  fn_apply_shared_kernel<IPT><<<(unsigned)blocks, 256, 0, St(stream)>>>(count, nterms, c, theta, coef,
                                                                      x, b, y, mode);
  FN_LAUNCHED();
  return 0;
}

int64_t rbws_fn_band_doubles(int count, int c, int planar) {
  const int64_t c1 = c + 1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : c1 * c1 * c1;
  return nsys * M * band_ws(band_w(c, planar));
}

int rbws_fn_band_factor(int count, int c, int planar, const double* coefA, double* band,
                        int* info, void* stream) {
  if (count <= 0 || c < 1 || !coefA || !band || !info)
    return rbws_set_error("rbws_fn_band_factor: bad argument", __FILE__, __LINE__);
  const int64_t c1 = c + 1, nodes = c1 * c1 * c1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : nodes;
  fn_band_build_kernel<<<grid_of(nodes, count), 256, 0, St(stream)>>>(count, c, planar, coefA, band);
  FN_LAUNCHED();
  const int w = band_w(c, planar);
  const size_t wsm = (size_t)(w + 2) * band_ws(w) * sizeof(double);
  static const int blk = [] {  // A/B: RBWS_BAND_FACTOR_BLK=0 keeps the row-by-row kernel
    const char* e = getenv("RBWS_BAND_FACTOR_BLK");
    return e ? atoi(e) : 1;
  }();
  constexpr int kNB = 16;
  const size_t bsm = (size_t)(w + kNB) * band_ws(w) * sizeof(double);
  if (blk && w < 256 && bsm <= 200 * 1024) {
    RBWS_CUDA_CHECK(rbws::smem_attr((const void*)band_factor_blk_kernel<kNB>, bsm));
    band_factor_blk_kernel<kNB><<<(unsigned)nsys, RBWS_BF_TPB, bsm, St(stream)>>>(nsys, M, w, band,
                                                                                 info);
  } else if (wsm <= 200 * 1024 && w < 32 * kFacK && !getenv("RBWS_BAND_FACTOR_GLOBAL")) {
    RBWS_CUDA_CHECK(rbws::smem_attr((const void*)band_factor_smem_kernel, wsm));
    band_factor_smem_kernel<<<(unsigned)nsys, 256, wsm, St(stream)>>>(nsys, M, w, band, info);
  } else {
    band_factor_kernel<<<(unsigned)nsys, 256, 0, St(stream)>>>(nsys, M, w, band, info);
  }
  FN_LAUNCHED();
  return 0;
}

static int band_solve_launch(int64_t nsys, int64_t M, int w, const double* band, int64_t lstride,
                             double* r, int64_t rstride, double* x, int64_t xstride, double omega,
                             int mode, cudaStream_t stream, bool allow_simple) {
  // sub-warp systems (LPS lanes each); RBWS_BAND_SOLVE_SIMPLE=1 for the warp-per-system
  // kernel (A/B, contiguous systems only)
  auto sub = [&](auto lps_c, auto kps_c) -> int {
    constexpr int LPS = decltype(lps_c)::value, KPS = decltype(kps_c)::value;
    constexpr int SPW = 32 / LPS;
    const int64_t warps_needed = (nsys + SPW - 1) / SPW;
    const unsigned nb = (unsigned)((warps_needed + 3) / 4);
    band_solve_sub_kernel<LPS, KPS, 4><<<nb, 128, 0, stream>>>(nsys, M, w, band, lstride, r, rstride,
                                                               x, xstride, omega, mode);
    FN_LAUNCHED();
    return 0;
  };
  // lanes per system: RBWS_BAND_LPS (8 / 16 / 32) for A/B
  static const int lps = getenv("RBWS_BAND_LPS") ? atoi(getenv("RBWS_BAND_LPS")) : 16;
  using std::integral_constant;
#define RBWS_SUB(L_, K_) \
  if (lps == L_ && w + 1 <= L_ * K_) return sub(integral_constant<int, L_>{}, integral_constant<int, K_>{});
  if (!(allow_simple && getenv("RBWS_BAND_SOLVE_SIMPLE"))) {
    RBWS_SUB(8, 1) RBWS_SUB(8, 2) RBWS_SUB(8, 3) RBWS_SUB(8, 5) RBWS_SUB(8, 9) RBWS_SUB(8, 17)
    RBWS_SUB(16, 1) RBWS_SUB(16, 2) RBWS_SUB(16, 3) RBWS_SUB(16, 5) RBWS_SUB(16, 9)
    RBWS_SUB(32, 1) RBWS_SUB(32, 2) RBWS_SUB(32, 3) RBWS_SUB(32, 5) RBWS_SUB(32, 9)
  }
#undef RBWS_SUB
  if (!allow_simple)
    return rbws_set_error("band solve: bandwidth beyond the sub-warp kernels", __FILE__, __LINE__);
  int ring = 32;
  while (ring < w + 1) ring *= 2;
  const int warps = 4;
  const size_t smem = (size_t)warps * ring * sizeof(double);
  if (smem > 48 * 1024) {
    RBWS_CUDA_CHECK(cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
  }
  band_solve_kernel<<<(unsigned)((nsys + warps - 1) / warps), warps * 32, smem, stream>>>(
      nsys, M, w, ring, band, r, x, omega, mode);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_band_solve(int count, int c, int planar, const double* band, double* r, double* x,
                       double omega, int mode, void* stream) {
  if (count <= 0 || c < 1 || !band || !r || !x || mode < 0 || mode > 1)
    return rbws_set_error("rbws_fn_band_solve: bad argument", __FILE__, __LINE__);
  const int64_t c1 = c + 1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : c1 * c1 * c1;
  const int w = band_w(c, planar);
  return band_solve_launch(nsys, M, w, band, M * band_ws(w), r, M, x, M, omega, mode, St(stream),
                           true);
}

int rbws_fn_band_transpose(int count, int c, int planar, const double* band, double* bandT,
                           void* stream) {
  if (count <= 0 || c < 1 || !band || !bandT)
    return rbws_set_error("rbws_fn_band_transpose: bad argument", __FILE__, __LINE__);
  const int64_t c1 = c + 1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : c1 * c1 * c1;
  const int w = band_w(c, planar);
  const int64_t tot = M * band_ws(w);
  dim3 grd((unsigned)((tot + 255) / 256), (unsigned)nsys);
  band_transpose_kernel<<<grd, 256, 0, St(stream)>>>(nsys, M, w, band, bandT);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_band_solve_t(int count, int c, int planar, const double* band, const double* bandT,
                         double* r, double* x, double omega, int mode, void* stream) {
  if (count <= 0 || c < 1 || !band || !bandT || !r || !x || mode < 0 || mode > 1)
    return rbws_set_error("rbws_fn_band_solve_t: bad argument", __FILE__, __LINE__);
  const int64_t c1 = c + 1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : c1 * c1 * c1;
  const int w = band_w(c, planar);
  const int sl = (w + 32 + 31) / 32;  // slots: w + 32 rows in flight
  const unsigned nb = (unsigned)((nsys + 3) / 4);
  const int64_t ls = M * band_ws(w);
#define RBWS_ROT(SL_)                                                                       \
  case SL_:                                                                                 \
    band_solve_rot_kernel<SL_><<<nb, 128, 0, St(stream)>>>(nsys, M, w, band, bandT, ls, r, M, \
                                                           x, M, omega, mode);              \
    break;
  switch (sl) {
    RBWS_ROT(2) RBWS_ROT(3) RBWS_ROT(4) RBWS_ROT(5) RBWS_ROT(6)
    default: return rbws_set_error("rbws_fn_band_solve_t: bandwidth beyond the kernels", __FILE__, __LINE__);
  }
#undef RBWS_ROT
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_plane_gs_sweep(int count, int c, const double* coefA, const double* band,
                           const double* b, double* x, double* scratch, int forward, void* stream) {
  if (count <= 0 || c < 1 || !coefA || !band || !b || !x || !scratch)
    return rbws_set_error("rbws_fn_plane_gs_sweep: bad argument", __FILE__, __LINE__);
  const int64_t c1 = c + 1, M = c1 * c1;
  const int w = band_w(c, 1);
  const int64_t lsz = M * band_ws(w);
  for (int q = 0; q <= c; ++q) {
    const int p = forward ? q : c - q;
    fn_plane_rhs_kernel<<<grid_of(M, count), 256, 0, St(stream)>>>(count, c, p, coefA, x, b, scratch);
    FN_LAUNCHED();
    // x_p = A_pp^-1 rhs for every instance: systems (i, p) at strides (c+1) planes
    if (band_solve_launch(count, M, w, band + p * lsz, c1 * lsz, scratch, M, x + p * M, c1 * M, 1.0,
                          0, St(stream), false))
      return 1;
  }
  return 0;
}

int rbws_fn_restrict(int count, int cc, const double* r_fine, double* b_coarse,
                     const unsigned char* coarse_mask, void* stream) {
  if (count <= 0 || cc < 1 || !r_fine || !b_coarse || !coarse_mask)
    return rbws_set_error("rbws_fn_restrict: bad argument", __FILE__, __LINE__);
  const int64_t cn = (int64_t)(cc + 1) * (cc + 1) * (cc + 1);
  fn_restrict_kernel<<<grid_of(cn, count), 256, 0, St(stream)>>>(count, cc, r_fine, b_coarse,
                                                                  coarse_mask);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_prolong_add(int count, int cc, const double* e_coarse, double* u_fine,
                        const unsigned char* fine_mask, void* stream) {
  if (count <= 0 || cc < 1 || !e_coarse || !u_fine || !fine_mask)
    return rbws_set_error("rbws_fn_prolong_add: bad argument", __FILE__, __LINE__);
  const int64_t fn = (int64_t)(2 * cc + 1) * (2 * cc + 1) * (2 * cc + 1);
  fn_prolong_kernel<<<grid_of(fn, count), 256, 0, St(stream)>>>(count, cc, e_coarse, u_fine, fine_mask);
  FN_LAUNCHED();
  return 0;
}

int rbws_fn_point_jacobi(int count, int c, const double* coefA, const double* r, double* x,
                         double omega, void* stream) {
  if (count <= 0 || c < 1 || !coefA || !r || !x)
    return rbws_set_error("rbws_fn_point_jacobi: bad argument", __FILE__, __LINE__);
  const int64_t nodes = (int64_t)(c + 1) * (c + 1) * (c + 1);
  fn_point_jacobi_kernel<<<grid_of(nodes, count), 256, 0, St(stream)>>>(count, nodes, coefA, r, x,
                                                                         omega);
  FN_LAUNCHED();
  return 0;
}

}  // extern "C"
