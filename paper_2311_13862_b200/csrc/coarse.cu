// Matrix-free coarse-level kernels (sm_100a).
//
// The Galerkin operator of level l is a sum of Kronecker products of 1D
// tridiagonal factors, one per affine term q and direction part d:
//   A_l(mu) = sum_q theta_q(mu) sum_d  Z_qd (x) Y_qd (x) X_qd,
// so its 27-point coefficient at node (I,J,K), offset (ox,oy,oz) is
//   c = sum_qd theta_q X_qd(I,I+ox) Y_qd(J,J+oy) Z_qd(K,K+oz).
// A thread owns a grid column (I,J) and marches in K.  The 27 coefficients
// are cached in registers and recomputed only on planes whose z factors differ
// from the previous plane's (a CTA-uniform flag); for thermal blocks that is
// a handful of planes per column, so per-instance coefficient arrays never
// exist in HBM.  The stencil input (tile rows + one halo row each side) and the
// centre rhs are staged with one TMA bulk copy per array per plane into an
// 8-slot mbarrier ring.
//
// The nu=1 pre-smoothing residual b - A(w D^-1 b) is evaluated as a plain
// residual of u = w D^-1 b, which the restriction kernel writes next to the
// coarse rhs (restrict_launch with dinv), so no per-neighbour scaling is needed.
#include "coarse.cuh"
#include "tma.cuh"

namespace rbws {

constexpr int kCStages = 8;
constexpr int kCMaxPlanes = 260;  // z-factor flag table bound (planes per z-chunk + 2)

// threads per CTA of the coarse-level kernels: 128 on grids up to 32 cells (four CTAs per SM
// hide the per-CTA weight set-up and the short z march better: coarse levels of configs[1]
// 0.91 -> 0.86 ms per V-cycle; 64 and 512 threads measured slower), 256 above
#ifndef RBWS_COARSE_SMALL_THREADS
#define RBWS_COARSE_SMALL_THREADS 128
#endif
CoarseGeom coarse_geom(int n, int batch, int nz) {
  CoarseGeom g;
  int ty = (n <= 32 ? RBWS_COARSE_SMALL_THREADS : 256) / n;
  if (ty < 1) ty = 1;
  if (ty > n) ty = n;
  g.ty = ty;
  g.threads = ty * n;
  g.ytiles = n / ty;
  if (nz <= 0) nz = n;
  g.zc = 1;
  while ((int64_t)g.ytiles * batch * g.zc < 2 * 148 && nz / (g.zc * 2) >= 8) g.zc *= 2;
  g.kz = (nz + g.zc - 1) / g.zc;
  return g;
}

struct CoarseArgs {
  int n, Q;
  const int* zsame;     // [n+1] plane k repeats plane k-1's z factors (host precomputed)
  const int* grp;       // [3Q] z-group of every term (kron kernel)
  CoarseGeom g;
  const double* fac;    // [Q*3][3][2][n+1]
  const double* theta;  // [batch][Q]
  const double* x;      // stencil input, staged with halo rows
  const double* b;      // centre rhs, staged (RESID / JACOBI)
  double* y;
  const int* active;
  double omega;
  int zlo, zhi;  // output planes [zlo, zhi) (global plane indices, virtual base pointers)
};

enum CoarseMode : int { CM_APPLY = 0, CM_RESID = 1, CM_JACOBI = 2, CM_PRE = 3, CM_DINV = 4 };

// T(i, i+o) of a 1D tridiagonal factor stored as [diag | upper] with stride n1
__device__ __forceinline__ double tri(const double* f, int n1, int i, int o) {
  if (o == 0) return __ldg(f + i);
  if (o > 0) return __ldg(f + n1 + i);
  return __ldg(f + n1 + i - 1);
}

template <int Q, int MODE>
__global__ void __launch_bounds__(256) coarse_kernel(CoarseArgs a) {
  constexpr int NH = (MODE == CM_DINV) ? 0 : 1;                          // halo-staged arrays
  constexpr int NC = (MODE == CM_RESID || MODE == CM_JACOBI) ? 1 : 0;     // centre-staged arrays
  constexpr int S = kCStages;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = a.n, n1 = n + 1;
  const int ty = a.g.ty, zc = a.g.zc;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (a.active && !a.active[mu]) return;
  const int j0 = blockIdx.y * ty;
  const int tid = threadIdx.x;
  const int64_t n2 = (int64_t)n * n;
  const int64_t base = (int64_t)mu * n2 * n;
  const int kz = a.g.kz;
  const int kb = max(1, a.zlo + kc * kz), ke = min(min(n, a.zhi), a.zlo + (kc + 1) * kz);
  if (kb >= ke) return;
  const int p_first = kb - 1, p_last = ke;
  const int np = p_last - p_first + 1;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int* zsame = reinterpret_cast<int*>(smem + 64);
  double* ring = reinterpret_cast<double*>(smem + 64 + 4 * kCMaxPlanes + 64);
  // slot = (ty+2) staged rows + 2 zero pad doubles: the 27-point corner neighbour of
  // the tile's last column/row reads one element past the staged rows (a ghost, 0)
  const int hsz = (ty + 2) * n + 2, csz = ty * n;
  const int ssz = NH * hsz + NC * csz;
  double* const xring = ring;
  auto xs = [&](int st) { return xring + st * ssz; };
  auto bs = [&](int st) { return xring + st * ssz + NH * hsz; };

  const double* fac = a.fac;
  const int fstride = 2 * n1;  // one axis factor [diag | upper]
  if (tid == 0 && NH > 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  if (NH > 0) {  // zero the pads and (first tile) the never-staged halo row above row 0
    for (int t = tid; t < S; t += blockDim.x) {
      xs(t)[hsz - 2] = 0.0;
      xs(t)[hsz - 1] = 0.0;
    }
    if (j0 == 0)
      for (int t = tid; t < S * n; t += blockDim.x) xs(t / n)[t % n] = 0.0;
  }
  for (int p = 1 + tid; p < np; p += blockDim.x) zsame[p] = a.zsame[p_first + p];
  __syncthreads();

  auto issue = [&](int p) {
    const int st = (p - p_first) & (S - 1);
    const int skip = (j0 == 0) ? 1 : 0;
    const uint32_t hbytes = (uint32_t)((ty + 2 - skip) * n * 8);
    const uint32_t cbytes = (uint32_t)(ty * n * 8);
    mbar_arrive_expect_tx(&bar[st], NH * hbytes + NC * cbytes);
    const int64_t plane = base + (int64_t)p * n2;
    bulk_g2s(xs(st) + skip * n, a.x + plane + (int64_t)(j0 - 1 + skip) * n, hbytes, &bar[st]);
    if (NC) bulk_g2s(bs(st), a.b + plane + (int64_t)j0 * n, cbytes, &bar[st]);
  };
  if (NH > 0 && tid == 0)
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);

  const int i = tid % n, jl = tid / n, j = j0 + jl;
  const bool on = (i >= 1) && (j >= 1);
  const double* th = a.theta + (size_t)mu * Q;
  // 27 coefficients c[(oz+1)*9 + (oy+1)*3 + (ox+1)]
  double c[27];
  auto coeffs = [&](int k) {
#pragma unroll
    for (int o = 0; o < 27; ++o) c[o] = 0.0;
    if (!on) return;
#pragma unroll
    for (int t = 0; t < 3 * Q; ++t) {
      const double tq = th[t / 3];
      const double* fx = fac + ((size_t)t * 3 + 0) * fstride;
      const double* fy = fac + ((size_t)t * 3 + 1) * fstride;
      const double* fz = fac + ((size_t)t * 3 + 2) * fstride;
      const double xv[3] = {tri(fx, n1, i, -1), tri(fx, n1, i, 0), tri(fx, n1, i, 1)};
      const double yv[3] = {tq * tri(fy, n1, j, -1), tq * tri(fy, n1, j, 0), tq * tri(fy, n1, j, 1)};
      const double zv[3] = {tri(fz, n1, k, -1), tri(fz, n1, k, 0), tri(fz, n1, k, 1)};
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const double yz = yv[dy] * zv[dz];
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) c[dz * 9 + dy * 3 + dx] = fma(xv[dx], yz, c[dz * 9 + dy * 3 + dx]);
        }
    }
  };

  const int hi = (jl + 1) * n + i;
  const double om = a.omega;
  double cdi = 0.0;
  // the 3x3 neighbourhood of this column in planes k-1, k, k+1 marches in registers:
  // each step reads only plane k+1's nine values from shared memory
  double va[9], vb[9], vcc[9];
  auto load9 = [&](int p, double* v) {
    const double* P = xs((p - p_first) & (S - 1)) + hi;
    v[0] = P[-n - 1]; v[1] = P[-n]; v[2] = P[-n + 1];
    v[3] = P[-1];     v[4] = P[0];  v[5] = P[1];
    v[6] = P[n - 1];  v[7] = P[n];  v[8] = P[n + 1];
  };
  auto wait = [&](int p) {
    const int t = p - p_first;
    mbar_wait(&bar[t & (S - 1)], (uint32_t)((t / S) & 1));
  };
  if (NH > 0) {
    wait(p_first);
    wait(p_first + 1);
    load9(p_first, va);
    load9(p_first + 1, vb);
  }
  // one node: down / centre / up neighbourhoods in registers
  auto step = [&](int k, const double* vd, const double* vc, double* vu) {
    if (k == kb || !zsame[k - p_first]) {
      coeffs(k);
      cdi = om / c[13];  // cached damping / diagonal (no per-node division)
    }
    const int64_t gidx = base + (int64_t)k * n2 + (int64_t)j * n + i;
    if (MODE == CM_DINV) {
      if (on) a.y[gidx] = 1.0 / c[13];
      return;
    }
    wait(k + 1);
    load9(k + 1, vu);
    double part[3];
    const double* V3[3] = {vd, vc, vu};
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
      const double* v = V3[dz];
      const double* cc = c + dz * 9;
      const double ra = fma(cc[2], v[2], fma(cc[1], v[1], cc[0] * v[0]));
      const double rb = fma(cc[5], v[5], fma(cc[4], v[4], cc[3] * v[3]));
      const double rc = fma(cc[8], v[8], fma(cc[7], v[7], cc[6] * v[6]));
      part[dz] = (ra + rb) + rc;
    }
    const double Au = (part[0] + part[2]) + part[1];
    if (on) {
      if (MODE == CM_APPLY) {
        a.y[gidx] = Au;
      } else if (MODE == CM_RESID) {
        a.y[gidx] = bs((k - p_first) & (S - 1))[jl * n + i] - Au;
      } else {  // CM_JACOBI
        const double bv = bs((k - p_first) & (S - 1))[jl * n + i];
        a.y[gidx] = fma(cdi, bv - Au, vc[4]);
      }
    }
  };
  // three planes per trip: the register roles rotate with period 3 (no moves)
  for (int k0 = kb; k0 < ke; k0 += 3) {
    step(k0, va, vb, vcc);
    if (k0 + 1 < ke) step(k0 + 1, vb, vcc, va);
    if (k0 + 2 < ke) step(k0 + 2, vcc, va, vb);
    if (NH > 0) {
      __syncthreads();  // every thread is done with planes <= k0+3
      if (tid == 0) {
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int pn = k0 - 1 + u + S;
          if (pn <= p_last) issue(pn);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// z-grouped Kronecker form (the fast path when few distinct z factors exist):
//   A = sum_g Z_g (x) W_g,   W_g = sum_{t in g} theta_t Y_t (x) X_t,
// so at node (I,J,K):  (A u) = sum_g sum_oz Z_g(K,oz) s_g(K+oz),
//   s_g(k) = sum_{ox,oy} W_g(I,J; ox,oy) u(I+ox, J+oy, k)   (9 FMAs per group).
// W_g (9G doubles) is plane-independent: computed once per CTA, never refreshed;
// s_g of planes k-1, k, k+1 march in registers; Z_g(k, .) is a CTA-uniform table.
// For thermal blocks G = 2 (4 with a z split): ~12G FMAs and 9 LDS per node and
// about a third of the 27-coefficient kernel's registers (two CTAs per SM).
// NT > 0: the grid size (and with it the tile rows, every shared-memory offset and row stride)
// is a compile-time constant — the generic kernel spends ~40 % of its instructions on index
// arithmetic (ncu: 149 instructions per node at 32^3, issue-bound); NT = 0: any grid.
__host__ __device__ constexpr int coarse_ty(int n) {
  return (n <= 32 ? RBWS_COARSE_SMALL_THREADS : 256) / n;
}
template <int G, int MODE, int NT = 0>
__global__ void __launch_bounds__(256, 2) coarse_kron_kernel(CoarseArgs a) {
  constexpr int NH = (MODE == CM_DINV) ? 0 : 1;
  constexpr int NC = (MODE == CM_RESID || MODE == CM_JACOBI) ? 1 : 0;
  constexpr int S = kCStages;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = NT > 0 ? NT : a.n, n1 = n + 1, Q = a.Q;
  const int ty = NT > 0 ? coarse_ty(NT > 0 ? NT : 1) : a.g.ty, zc = a.g.zc;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (a.active && !a.active[mu]) return;
  const int j0 = blockIdx.y * ty;
  const int tid = threadIdx.x;
  const int64_t n2 = (int64_t)n * n;
  const int64_t base = (int64_t)mu * n2 * n;
  const int kz = a.g.kz;
  const int kb = max(1, a.zlo + kc * kz), ke = min(min(n, a.zhi), a.zlo + (kc + 1) * kz);
  if (kb >= ke) return;
  const int p_first = kb - 1, p_last = ke;
  const int np = p_last - p_first + 1;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int* zdsame = reinterpret_cast<int*>(smem + 64);                      // [kCMaxPlanes]
  double* zg = reinterpret_cast<double*>(smem + 64 + 4 * kCMaxPlanes);   // [np][G][3]
  double* ring = zg + ((np * G * 3 + 1) & ~1);
  const int hsz = (ty + 2) * n + 2, csz = ty * n;
  const int ssz = NH * hsz + NC * csz;
  auto xs = [&](int st) { return ring + st * ssz; };
  auto bs = [&](int st) { return ring + st * ssz + NH * hsz; };
  const double* fac = a.fac;
  const int fstride = 2 * n1;

  if (tid == 0 && NH > 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  if (NH > 0) {  // zero the pads and (first tile) the never-staged halo row above row 0
    for (int t = tid; t < S; t += blockDim.x) {
      xs(t)[hsz - 2] = 0.0;
      xs(t)[hsz - 1] = 0.0;
    }
    if (j0 == 0)
      for (int t = tid; t < S * n; t += blockDim.x) xs(t / n)[t % n] = 0.0;
  }
  // z stencil of every group at every staged plane (from the group's first term)
  for (int t = tid; t < np * G * 3; t += blockDim.x) {
    const int p = t / (3 * G), g = (t / 3) % G, o = t % 3 - 1, k = p_first + p;
    int rep = 0;
    for (int u = 3 * Q - 1; u >= 0; --u)
      if (a.grp[u] == g) rep = u;
    const double* fz = fac + ((size_t)rep * 3 + 2) * fstride;
    zg[t] = (k >= 1 && k <= n - 1) ? tri(fz, n1, k, o) : 0.0;
  }
  __syncthreads();
  for (int p = 1 + tid; p < np; p += blockDim.x) {  // diagonal z entries repeat plane p-1's?
    int same = 1;
    for (int g = 0; g < G; ++g) same &= (zg[(p * G + g) * 3 + 1] == zg[((p - 1) * G + g) * 3 + 1]);
    zdsame[p] = same;
  }

  auto issue = [&](int p) {
    const int st = (p - p_first) & (S - 1);
    const int skip = (j0 == 0) ? 1 : 0;
    const uint32_t hbytes = (uint32_t)((ty + 2 - skip) * n * 8);
    const uint32_t cbytes = (uint32_t)(ty * n * 8);
    mbar_arrive_expect_tx(&bar[st], NH * hbytes + NC * cbytes);
    const int64_t plane = base + (int64_t)p * n2;
    bulk_g2s(xs(st) + skip * n, a.x + plane + (int64_t)(j0 - 1 + skip) * n, hbytes, &bar[st]);
    if (NC) bulk_g2s(bs(st), a.b + plane + (int64_t)j0 * n, cbytes, &bar[st]);
  };
  if (NH > 0 && tid == 0)
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);

  const int i = tid % n, jl = tid / n, j = j0 + jl;
  const bool on = (i >= 1) && (j >= 1);
  const double* th = a.theta + (size_t)mu * Q;
  // W_g(ox, oy) of this column, w[g*9 + (oy+1)*3 + (ox+1)]
  double w[G * 9];
#pragma unroll
  for (int o = 0; o < G * 9; ++o) w[o] = 0.0;
  if (on) {
    for (int t = 0; t < 3 * Q; ++t) {
      const int gt = __ldg(a.grp + t);
      const double tq = th[t / 3];
      const double* fx = fac + ((size_t)t * 3 + 0) * fstride;
      const double* fy = fac + ((size_t)t * 3 + 1) * fstride;
      const double xv[3] = {tri(fx, n1, i, -1), tri(fx, n1, i, 0), tri(fx, n1, i, 1)};
      const double yv[3] = {tq * tri(fy, n1, j, -1), tq * tri(fy, n1, j, 0), tq * tri(fy, n1, j, 1)};
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (gt == g) {
#pragma unroll
          for (int oy = 0; oy < 3; ++oy)
#pragma unroll
            for (int ox = 0; ox < 3; ++ox) w[g * 9 + oy * 3 + ox] = fma(yv[oy], xv[ox], w[g * 9 + oy * 3 + ox]);
        }
    }
  }
  __syncthreads();  // zdsame visible

  const int hi = (jl + 1) * n + i;
  const double om = a.omega;
  double cdi = 0.0, dg = 0.0;
  auto wait = [&](int p) {
    const int t = p - p_first;
    mbar_wait(&bar[t & (S - 1)], (uint32_t)((t / S) & 1));
  };
  // s_g of one staged plane; centre value returned in xc
  auto conv = [&](int p, double* s, double& xc) {
    const double* P = xs((p - p_first) & (S - 1)) + hi;
    const double v[9] = {P[-n - 1], P[-n], P[-n + 1], P[-1], P[0], P[1], P[n - 1], P[n], P[n + 1]};
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double* wg = w + g * 9;
      const double ra = fma(wg[2], v[2], fma(wg[1], v[1], wg[0] * v[0]));
      const double rb = fma(wg[5], v[5], fma(wg[4], v[4], wg[3] * v[3]));
      const double rc = fma(wg[8], v[8], fma(wg[7], v[7], wg[6] * v[6]));
      s[g] = (ra + rb) + rc;
    }
    xc = v[4];
  };
  double sa[G], sb[G], sc[G], xa = 0.0, xb = 0.0, xcv = 0.0;
  if (NH > 0) {
    wait(p_first);
    wait(p_first + 1);
    conv(p_first, sa, xa);
    conv(p_first + 1, sb, xb);
  }
  auto step = [&](int k, const double* sd, const double* s0, double* su, double x0, double& xu) {
    const double* zk = zg + (k - p_first) * G * 3;
    if (MODE == CM_DINV || MODE == CM_JACOBI) {
      if (k == kb || !zdsame[k - p_first]) {
        dg = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) dg = fma(zk[g * 3 + 1], w[g * 9 + 4], dg);
        cdi = om / dg;  // cached damping / diagonal (no per-node division)
      }
    }
    const int64_t gidx = base + (int64_t)k * n2 + (int64_t)j * n + i;
    if (MODE == CM_DINV) {
      if (on) a.y[gidx] = 1.0 / dg;
      return;
    }
    wait(k + 1);
    conv(k + 1, su, xu);
    double Au = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g)
      Au = fma(zk[g * 3 + 0], sd[g], fma(zk[g * 3 + 1], s0[g], fma(zk[g * 3 + 2], su[g], Au)));
    if (on) {
      if (MODE == CM_APPLY) {
        a.y[gidx] = Au;
      } else if (MODE == CM_RESID) {
        a.y[gidx] = bs((k - p_first) & (S - 1))[jl * n + i] - Au;
      } else {  // CM_JACOBI
        const double bv = bs((k - p_first) & (S - 1))[jl * n + i];
        a.y[gidx] = fma(cdi, bv - Au, x0);
      }
    }
  };
  // three planes per trip: the register roles rotate with period 3 (no moves)
  for (int k0 = kb; k0 < ke; k0 += 3) {
    step(k0, sa, sb, sc, xb, xcv);
    if (k0 + 1 < ke) step(k0 + 1, sb, sc, sa, xcv, xa);
    if (k0 + 2 < ke) step(k0 + 2, sc, sa, sb, xa, xb);
    if (NH > 0) {
      __syncthreads();  // every thread is done with planes <= k0+3
      if (tid == 0) {
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int pn = k0 - 1 + u + S;
          if (pn <= p_last) issue(pn);
        }
      }
    }
  }
}

template <int G, int MODE>
static cudaError_t coarse_kron_launch_m(CoarseArgs a, int batch, cudaStream_t stream) {
  constexpr int NH = (MODE == CM_DINV) ? 0 : 1;
  constexpr int NC = (MODE == CM_RESID || MODE == CM_JACOBI) ? 1 : 0;
  a.g = coarse_geom(a.n, batch, a.zhi - a.zlo);
  const int np = a.g.kz + 2;
  if (np > kCMaxPlanes) return cudaErrorInvalidValue;
  const size_t smem = 64 + 4 * kCMaxPlanes + 8 * (((size_t)np * G * 3 + 1) & ~(size_t)1) +
                      (size_t)kCStages * (NH * ((a.g.ty + 2) * a.n + 2) + NC * a.g.ty * a.n) * 8;
  dim3 grd(1, a.g.ytiles, batch * a.g.zc);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    count_launch();
    kern<<<grd, a.g.threads, smem, stream>>>(a);
    return cudaGetLastError();
  };
  // compile-time grid size for the sizes of the BASELINE hierarchies (RESID / JACOBI: the
  // V-cycle's kernels)
  if (MODE == CM_RESID || MODE == CM_JACOBI) {
    if (a.n == 16 && a.g.ty == coarse_ty(16)) return go(coarse_kron_kernel<G, MODE, 16>);
    if (a.n == 32 && a.g.ty == coarse_ty(32)) return go(coarse_kron_kernel<G, MODE, 32>);
    if (a.n == 64 && a.g.ty == coarse_ty(64)) return go(coarse_kron_kernel<G, MODE, 64>);
  }
  return go(coarse_kron_kernel<G, MODE, 0>);
}

template <int G>
static cudaError_t coarse_kron_launch_g(int mode, const CoarseArgs& a, int batch,
                                        cudaStream_t stream) {
  switch (mode) {
    case CM_APPLY: return coarse_kron_launch_m<G, CM_APPLY>(a, batch, stream);
    case CM_RESID: return coarse_kron_launch_m<G, CM_RESID>(a, batch, stream);
    case CM_JACOBI: return coarse_kron_launch_m<G, CM_JACOBI>(a, batch, stream);
    case CM_DINV: return coarse_kron_launch_m<G, CM_DINV>(a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q, int MODE>
static cudaError_t coarse_launch_m(CoarseArgs a, int batch, cudaStream_t stream) {
  constexpr int NH = (MODE == CM_DINV) ? 0 : 1;
  constexpr int NC = (MODE == CM_RESID || MODE == CM_JACOBI) ? 1 : 0;
  a.g = coarse_geom(a.n, batch, a.zhi - a.zlo);
  if (a.g.kz + 2 > kCMaxPlanes) return cudaErrorInvalidValue;
  const size_t smem = 64 + 4 * kCMaxPlanes + 64 +
                      (size_t)kCStages * (NH * ((a.g.ty + 2) * a.n + 2) + NC * a.g.ty * a.n) * 8;
  {
    cudaError_t e = smem_attr((const void*)coarse_kernel<Q, MODE>, smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd(1, a.g.ytiles, batch * a.g.zc);
  count_launch();
  coarse_kernel<Q, MODE><<<grd, a.g.threads, smem, stream>>>(a);
  return cudaGetLastError();
}

template <int Q>
static cudaError_t coarse_launch_q(int mode, const CoarseArgs& a, int batch, cudaStream_t stream) {
  switch (mode) {
    case CM_APPLY: return coarse_launch_m<Q, CM_APPLY>(a, batch, stream);
    case CM_RESID: return coarse_launch_m<Q, CM_RESID>(a, batch, stream);
    case CM_JACOBI: return coarse_launch_m<Q, CM_JACOBI>(a, batch, stream);
    case CM_DINV: return coarse_launch_m<Q, CM_DINV>(a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ---- stored 27-point coefficients (levels with many z-groups) ---------------------
// The 13 forward offsets (dx, dy, dz), (dz, dy, dx) lexicographically positive; the
// backward coefficient of node X for -o is the forward one of node X - o (symmetry).
__device__ __forceinline__ void fwd_off(int o, int& dx, int& dy, int& dz) {
  const int t = o - 1;
  if (t < 9) { dz = 1; dy = t / 3 - 1; dx = t % 3 - 1; }
  else if (t < 12) { dz = 0; dy = 1; dx = t - 10; }
  else { dz = 0; dy = 0; dx = 1; }
}

__global__ void __launch_bounds__(256) coarse_build_kernel(int n, int Q,
                                                           const double* __restrict__ fac,
                                                           const double* __restrict__ theta,
                                                           double* __restrict__ coef,
                                                           double* __restrict__ dinv) {
  const int mu = blockIdx.y;
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const int i = X % n, j = (X / n) % n, k = (int)(X / ((int64_t)n * n));
  double* C = coef + (int64_t)mu * 14 * n3;
  const bool ghost = (i == 0 || j == 0 || k == 0);
  const int n1 = n + 1;
  // per term: the 3x3x3 factor values of each part loaded once (9 loads per part),
  // s[o] = sum_d fx fy fz, then c[o] += theta_q s[o] (the summation order of the
  // per-offset formulation)
  double c[14];
#pragma unroll
  for (int o = 0; o < 14; ++o) c[o] = 0.0;
  if (!ghost) {
    for (int q = 0; q < Q; ++q) {
      double sq[14];
#pragma unroll
      for (int o = 0; o < 14; ++o) sq[o] = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double* f = fac + (size_t)((q * 3 + d) * 3) * 2 * n1;
        double fx[3], fy[3], fz[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          fx[t] = tri(f, n1, i, t - 1);
          fy[t] = tri(f + 2 * n1, n1, j, t - 1);
          fz[t] = tri(f + 4 * n1, n1, k, t - 1);
        }
#pragma unroll
        for (int o = 0; o < 14; ++o) {
          int dx = 0, dy = 0, dz = 0;
          if (o > 0) fwd_off(o, dx, dy, dz);
          sq[o] += fx[dx + 1] * fy[dy + 1] * fz[dz + 1];
        }
      }
      const double t = theta[(int64_t)mu * Q + q];
#pragma unroll
      for (int o = 0; o < 14; ++o) c[o] = fma(t, sq[o], c[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < 14; ++o) C[o * n3 + X] = c[o];
  const double c0 = c[0];
  dinv[(int64_t)mu * n3 + X] = ghost ? 0.0 : 1.0 / c0;
}

cudaError_t coarse_build_coef(const CoarseOp& op, const double* theta, int batch, double* coef,
                              double* dinv, cudaStream_t stream) {
  const int64_t n3 = (int64_t)op.n * op.n * op.n;
  dim3 grd((unsigned)((n3 + 255) / 256), batch);
  count_launch();
  coarse_build_kernel<<<grd, 256, 0, stream>>>(op.n, op.Q, op.fac, theta, coef, dinv);
  return cudaGetLastError();
}

// one node per thread over the planes [zlo, zhi); coefficients streamed, neighbours
// through L1/L2.  mode: 0 y = A x, 1 y = b - A x, 2 y = x + w (b - A x)/diag, 4 y = 1/diag
template <int MODE>
__global__ void __launch_bounds__(256) coarse_stored_kernel(int n, const double* __restrict__ coef,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ y,
                                                            const int* __restrict__ active,
                                                            double omega, int zlo, int zhi,
                                                            int64_t cstride) {
  const int mu = blockIdx.y;
  if (active && !active[mu]) return;
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
  const int64_t X = (int64_t)zlo * n2 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= (int64_t)zhi * n2) return;
  const int i = X % n, j = (X / n) % n, k = (int)(X / n2);
  if (i == 0 || j == 0 || k == 0) return;
  const double* C = coef + (int64_t)mu * cstride;
  const int64_t base = (int64_t)mu * n3;
  const double c0 = __ldg(C + X);
  if (MODE == 4) {
    y[base + X] = 1.0 / c0;
    return;
  }
  const double* xb = x + base;
  const double xc = __ldg(xb + X);
  double Au = c0 * xc;
#pragma unroll
  for (int o = 1; o < 14; ++o) {
    int dx, dy, dz;
    fwd_off(o, dx, dy, dz);
    const int64_t off = dx + (int64_t)n * (dy + (int64_t)n * dz);
    Au = fma(__ldg(C + o * n3 + X), __ldg(xb + X + off), Au);
    Au = fma(__ldg(C + o * n3 + X - off), __ldg(xb + X - off), Au);
  }
  double out;
  if (MODE == 0) out = Au;
  else if (MODE == 1) out = __ldg(b + base + X) - Au;
  else out = fma(omega / c0, __ldg(b + base + X) - Au, xc);
  y[base + X] = out;
}

static cudaError_t coarse_stored_launch(int mode, const CoarseOp& op, int batch, const double* x,
                                        const double* b, double* y, double omega,
                                        const LaunchCtx& lc) {
  const int n = op.n;
  const int zlo = lc.zhi > 0 ? lc.zlo : 0, zhi = lc.zhi > 0 ? lc.zhi : n;
  const int64_t cnt = (int64_t)(zhi - zlo) * n * n;
  dim3 grd((unsigned)((cnt + 255) / 256), batch);
  const int64_t cs = op.coef_shared ? 0 : (int64_t)14 * n * n * n;
  count_launch();
  switch (mode) {
    case 0: coarse_stored_kernel<0><<<grd, 256, 0, lc.stream>>>(n, op.coef, x, b, y, lc.active, omega, zlo, zhi, cs); break;
    case 1: coarse_stored_kernel<1><<<grd, 256, 0, lc.stream>>>(n, op.coef, x, b, y, lc.active, omega, zlo, zhi, cs); break;
    case 2: coarse_stored_kernel<2><<<grd, 256, 0, lc.stream>>>(n, op.coef, x, b, y, lc.active, omega, zlo, zhi, cs); break;
    case 4: coarse_stored_kernel<4><<<grd, 256, 0, lc.stream>>>(n, op.coef, x, b, y, lc.active, omega, zlo, zhi, cs); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ---- per-term coefficients shared by the batch (assembled problems, finest level) ----------
// The batch's operators differ only in theta: a thread owns one node and IB instances, loads
// each per-term coefficient once and combines it for all IB instances (the combination order
// of stored_combine, the accumulation order of coarse_stored_kernel: bitwise the same
// results).  Instance groups are the fastest grid dimension, so the CTAs resident at one time
// work on the same nodes and the term coefficients are L2 hits after the first group: per
// node and instance HBM sees only the vectors.
#ifndef RBWS_SHARED_MINB
#define RBWS_SHARED_MINB 2
#endif
#ifndef RBWS_SHARED_UNROLL
#define RBWS_SHARED_UNROLL 13
#endif
#define RBWS_PRAGMA(x) _Pragma(#x)
#define RBWS_UNROLL(n) RBWS_PRAGMA(unroll n)
template <int MODE, int Q, int IB>
__global__ void __launch_bounds__(256, RBWS_SHARED_MINB) stored_shared_kernel(int n, int batch,
                                                            const double* __restrict__ tc,
                                                            const double* __restrict__ theta,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ y,
                                                            const int* __restrict__ active,
                                                            double omega, int zlo, int zhi) {
  const int mu0 = blockIdx.x * IB;
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
  const int64_t X = (int64_t)zlo * n2 + (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (X >= (int64_t)zhi * n2) return;
  const int i = X % n, j = (X / n) % n, k = (int)(X / n2);
  if (i == 0 || j == 0 || k == 0) return;
  bool on[IB];
  double th[IB][Q];
  int nact = 0;
#pragma unroll
  for (int u = 0; u < IB; ++u) {
    const int mu = mu0 + u;
    on[u] = mu < batch && (!active || active[mu]);
    nact += on[u] ? 1 : 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) th[u][q] = on[u] ? __ldg(theta + (int64_t)mu * Q + q) : 0.0;
  }
  if (!nact) return;
  auto comb = [&](const double* cq, int u) {  // sum_q theta_q c_q in stored_combine's order
    double v = th[u][0] * cq[0];
#pragma unroll
    for (int q = 1; q < Q; ++q) v = fma(th[u][q], cq[q], v);
    return v;
  };
  double cq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) cq[q] = __ldg(tc + (int64_t)q * 14 * n3 + X);
  double acc[IB], c0[IB], xc[IB];
#pragma unroll
  for (int u = 0; u < IB; ++u) {
    c0[u] = comb(cq, u);
    xc[u] = on[u] ? __ldg(x + (int64_t)(mu0 + u) * n3 + X) : 0.0;
    acc[u] = c0[u] * xc[u];
  }
  RBWS_UNROLL(RBWS_SHARED_UNROLL)
  for (int o = 1; o < 14; ++o) {
    int dx, dy, dz;
    fwd_off(o, dx, dy, dz);
    const int64_t off = dx + (int64_t)n * (dy + (int64_t)n * dz);
    double cf[Q], cb[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      cf[q] = __ldg(tc + ((int64_t)q * 14 + o) * n3 + X);
      cb[q] = __ldg(tc + ((int64_t)q * 14 + o) * n3 + X - off);
    }
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      if (!on[u]) continue;
      const double* xb = x + (int64_t)(mu0 + u) * n3;
      acc[u] = fma(comb(cf, u), __ldg(xb + X + off), acc[u]);
      acc[u] = fma(comb(cb, u), __ldg(xb + X - off), acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < IB; ++u) {
    if (!on[u]) continue;
    const int64_t o = (int64_t)(mu0 + u) * n3 + X;
    double out;
    if (MODE == 0) out = acc[u];
    else if (MODE == 1) out = __ldg(b + o) - acc[u];
    else out = fma(omega / c0[u], __ldg(b + o) - acc[u], xc[u]);
    y[o] = out;
  }
}

template <int Q, int IB>
static cudaError_t stored_shared_launch_qi(int mode, const CoarseOp& op, const double* theta,
                                           int batch, const double* x, const double* b,
                                           double* y, double omega, const LaunchCtx& lc) {
  const int n = op.n;
  const int zlo = lc.zhi > 0 ? lc.zlo : 0, zhi = lc.zhi > 0 ? lc.zhi : n;
  const int64_t cnt = (int64_t)(zhi - zlo) * n * n;
  dim3 grd((unsigned)((batch + IB - 1) / IB), (unsigned)((cnt + 255) / 256));
  count_launch();
#define RBWS_SSK(M) stored_shared_kernel<M, Q, IB><<<grd, 256, 0, lc.stream>>>( \
    n, batch, op.tcoef, theta, x, b, y, lc.active, omega, zlo, zhi)
  switch (mode) {
    case 0: RBWS_SSK(0); break;
    case 1: RBWS_SSK(1); break;
    case 2: RBWS_SSK(2); break;
    default: return cudaErrorInvalidValue;
  }
#undef RBWS_SSK
  return cudaGetLastError();
}

// instances per thread (RBWS_FEM_IB = 2 | 4 | 8 for A/B runs)
template <int Q>
static cudaError_t stored_shared_launch_q(int mode, const CoarseOp& op, const double* theta,
                                          int batch, const double* x, const double* b, double* y,
                                          double omega, const LaunchCtx& lc) {
  static const int ib = [] {
    const char* e = getenv("RBWS_FEM_IB");
    return e ? atoi(e) : 4;
  }();
  if (ib == 2) return stored_shared_launch_qi<Q, 2>(mode, op, theta, batch, x, b, y, omega, lc);
  if (ib == 8) return stored_shared_launch_qi<Q, 8>(mode, op, theta, batch, x, b, y, omega, lc);
  return stored_shared_launch_qi<Q, 4>(mode, op, theta, batch, x, b, y, omega, lc);
}

static cudaError_t stored_shared_launch(int mode, const CoarseOp& op, const double* theta,
                                        int batch, const double* x, const double* b, double* y,
                                        double omega, const LaunchCtx& lc) {
  switch (op.Q) {
    case 1: return stored_shared_launch_q<1>(mode, op, theta, batch, x, b, y, omega, lc);
    case 2: return stored_shared_launch_q<2>(mode, op, theta, batch, x, b, y, omega, lc);
    case 3: return stored_shared_launch_q<3>(mode, op, theta, batch, x, b, y, omega, lc);
    case 4: return stored_shared_launch_q<4>(mode, op, theta, batch, x, b, y, omega, lc);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t coarse_launch(int mode, const CoarseOp& op, const double* theta, int batch,
                          const double* x, const double* b, double* y, double omega,
                          const LaunchCtx& lc) {
  if (op.coef) return coarse_stored_launch(mode, op, batch, x, b, y, omega, lc);
  if (op.tcoef) {
    if (mode <= 2 && stored_zm_ok(op.n, op.Q, lc))
      return stored_zm_launch(mode, op.n, op.Q, op.tcoef, theta, op.dinv, batch, x, b, y, omega,
                              lc);
    return stored_shared_launch(mode, op, theta, batch, x, b, y, omega, lc);
  }
  const int n = op.n;
  if (n < 2 || n > 256) return cudaErrorInvalidValue;
  CoarseArgs a{};
  a.n = n;
  a.Q = op.Q;
  a.zsame = op.zsame;
  a.grp = op.grp;
  a.fac = op.fac;
  a.theta = theta;
  a.x = x;
  a.b = b;
  a.y = y;
  a.active = lc.active;
  a.omega = omega;
  a.zlo = lc.zhi > 0 ? lc.zlo : 0;
  a.zhi = lc.zhi > 0 ? lc.zhi : n;
  switch (op.G) {  // few z-groups: grouped Kronecker kernel
    case 1: return coarse_kron_launch_g<1>(mode, a, batch, lc.stream);
    case 2: return coarse_kron_launch_g<2>(mode, a, batch, lc.stream);
    case 3: return coarse_kron_launch_g<3>(mode, a, batch, lc.stream);
    case 4: return coarse_kron_launch_g<4>(mode, a, batch, lc.stream);
    default: break;
  }
  switch (op.Q) {  // general: 27 register coefficients per column
    case 1: return coarse_launch_q<1>(mode, a, batch, lc.stream);
    case 2: return coarse_launch_q<2>(mode, a, batch, lc.stream);
    case 3: return coarse_launch_q<3>(mode, a, batch, lc.stream);
    case 4: return coarse_launch_q<4>(mode, a, batch, lc.stream);
    case 5: return coarse_launch_q<5>(mode, a, batch, lc.stream);
    case 6: return coarse_launch_q<6>(mode, a, batch, lc.stream);
    case 7: return coarse_launch_q<7>(mode, a, batch, lc.stream);
    case 8: return coarse_launch_q<8>(mode, a, batch, lc.stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbws

namespace rbws {

// ---------------------------------------------------------------- coarsest level
// right-looking Cholesky of the m x m matrix A (shared memory, lower triangle) by the whole
// CTA; L (global) gets the factor, *status 1 if a pivot was not positive
__device__ void chol_store(double* A, int m, double* L, int* status) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < m; ++c) {
    if (threadIdx.x == 0) {
      const double dd = A[c * m + c];
      if (!(dd > 0.0)) bad = 1;
      A[c * m + c] = sqrt(dd > 0.0 ? dd : 1.0);
    }
    __syncthreads();
    const double piv = A[c * m + c];
    for (int r = c + 1 + threadIdx.x; r < m; r += blockDim.x) A[r * m + c] /= piv;
    __syncthreads();
    for (int t = threadIdx.x; t < (m - c - 1) * (m - c - 1); t += blockDim.x) {
      const int r = c + 1 + t / (m - c - 1), s = c + 1 + t % (m - c - 1);
      if (s <= r) A[r * m + s] -= A[r * m + c] * A[s * m + c];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int r = t / m, s = t % m;
    L[t] = (s <= r) ? A[t] : 0.0;
  }
  if (threadIdx.x == 0 && status) *status = bad;
}

// Dense Galerkin operator of the coarsest level assembled from the Kronecker
// factors, then Cholesky-factored in shared memory (one CTA per instance).
__global__ void coarse_factor_kf_kernel(int n0, int Q, const double* __restrict__ fac,
                                        const double* __restrict__ theta,
                                        double* __restrict__ Lout, int* __restrict__ status) {
  extern __shared__ double A[];
  const int m1 = n0 - 1, m = m1 * m1 * m1, n1 = n0 + 1, fstride = 2 * n1;
  const int mu = blockIdx.x;
  const double* th = theta + (size_t)mu * Q;
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int r = t / m, cidx = t % m;
    const int i = r % m1 + 1, j = (r / m1) % m1 + 1, k = r / (m1 * m1) + 1;
    const int i2 = cidx % m1 + 1, j2 = (cidx / m1) % m1 + 1, k2 = cidx / (m1 * m1) + 1;
    const int ox = i2 - i, oy = j2 - j, oz = k2 - k;
    double v = 0.0;
    if (ox >= -1 && ox <= 1 && oy >= -1 && oy <= 1 && oz >= -1 && oz <= 1) {
      for (int p = 0; p < 3 * Q; ++p) {
        const double* f = fac + (size_t)p * 3 * fstride;
        v = fma(th[p / 3], tri(f, n1, i, ox) * tri(f + fstride, n1, j, oy) *
                               tri(f + 2 * fstride, n1, k, oz), v);
      }
    }
    A[t] = v;
  }
  __syncthreads();
  chol_store(A, m, Lout + (int64_t)mu * m * m, status ? status + mu : nullptr);
}

cudaError_t coarse_factor_kf(int n0, int Q, const double* fac, const double* theta, int batch,
                             double* L, int* status, cudaStream_t stream) {
  const int m1 = n0 - 1, m = m1 * m1 * m1;
  const size_t smem = (size_t)m * m * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(coarse_factor_kf_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  coarse_factor_kf_kernel<<<batch, 128, smem, stream>>>(n0, Q, fac, theta, L, status);
  return cudaGetLastError();
}

}  // namespace rbws

namespace rbws {

// ---------------------------------------------------------------- stored-coefficient hierarchy
// (assembled FEM problems): per-term coefficients are mu-independent, the per-instance
// operator of a level is their theta-weighted sum in term order (reference grid.py:246-255)
__global__ void __launch_bounds__(256) stored_combine_kernel(int n, int Q,
                                                             const double* __restrict__ tcoef,
                                                             const double* __restrict__ theta,
                                                             double* __restrict__ coef,
                                                             double* __restrict__ dinv) {
  const int mu = blockIdx.y;
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const double* th = theta + (int64_t)mu * Q;
  double c0 = 0.0;
  const int no = coef ? 14 : 1;
  for (int o = 0; o < no; ++o) {
    double v = th[0] * __ldg(tcoef + o * n3 + X);
    for (int q = 1; q < Q; ++q) v = fma(th[q], __ldg(tcoef + ((int64_t)q * 14 + o) * n3 + X), v);
    if (coef) coef[(int64_t)mu * 14 * n3 + o * n3 + X] = v;
    if (o == 0) c0 = v;
  }
  const int i = X % n, j = (X / n) % n, k = (int)(X / ((int64_t)n * n));
  dinv[(int64_t)mu * n3 + X] = (i == 0 || j == 0 || k == 0) ? 0.0 : 1.0 / c0;
}

cudaError_t stored_combine(int n, int Q, const double* tcoef, const double* theta, int batch,
                           double* coef, double* dinv, cudaStream_t stream) {
  const int64_t n3 = (int64_t)n * n * n;
  dim3 grd((unsigned)((n3 + 255) / 256), batch);
  count_launch();
  stored_combine_kernel<<<grd, 256, 0, stream>>>(n, Q, tcoef, theta, coef, dinv);
  return cudaGetLastError();
}

__device__ __forceinline__ int fwd_index(int dx, int dy, int dz) {
  // inverse of fwd_off for a lexicographically positive offset
  if (dz == 1) return 1 + (dy + 1) * 3 + (dx + 1);
  if (dy == 1) return 10 + (dx + 1);
  return 13;
}

__global__ void coarse_factor_stored_kernel(int n0, int Q, const double* __restrict__ tcoef,
                                            const double* __restrict__ theta,
                                            double* __restrict__ Lout, int* __restrict__ status) {
  extern __shared__ double A[];
  const int m1 = n0 - 1, m = m1 * m1 * m1;
  const int64_t n3 = (int64_t)n0 * n0 * n0;
  const int mu = blockIdx.x;
  const double* th = theta + (size_t)mu * Q;
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int r = t / m, cidx = t % m;
    const int i = r % m1 + 1, j = (r / m1) % m1 + 1, k = r / (m1 * m1) + 1;
    const int i2 = cidx % m1 + 1, j2 = (cidx / m1) % m1 + 1, k2 = cidx / (m1 * m1) + 1;
    int ox = i2 - i, oy = j2 - j, oz = k2 - k;
    double v = 0.0;
    if (ox >= -1 && ox <= 1 && oy >= -1 && oy <= 1 && oz >= -1 && oz <= 1) {
      // the coefficient is stored at the row whose offset to the other node is forward
      int64_t X = i + (int64_t)n0 * (j + (int64_t)n0 * k);
      int o = 0;
      if (ox || oy || oz) {
        const bool fwd = oz > 0 || (oz == 0 && (oy > 0 || (oy == 0 && ox > 0)));
        if (!fwd) {
          X = i2 + (int64_t)n0 * (j2 + (int64_t)n0 * k2);
          ox = -ox; oy = -oy; oz = -oz;
        }
        o = fwd_index(ox, oy, oz);
      }
      v = th[0] * tcoef[o * n3 + X];
      for (int q = 1; q < Q; ++q) v = fma(th[q], tcoef[((int64_t)q * 14 + o) * n3 + X], v);
    }
    A[t] = v;
  }
  __syncthreads();
  chol_store(A, m, Lout + (int64_t)mu * m * m, status ? status + mu : nullptr);
}

cudaError_t coarse_factor_stored(int n0, int Q, const double* tcoef, const double* theta,
                                 int batch, double* L, int* status, cudaStream_t stream) {
  const int m1 = n0 - 1, m = m1 * m1 * m1;
  const size_t smem = (size_t)m * m * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(coarse_factor_stored_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  coarse_factor_stored_kernel<<<batch, 128, smem, stream>>>(n0, Q, tcoef, theta, L, status);
  return cudaGetLastError();
}

}  // namespace rbws
