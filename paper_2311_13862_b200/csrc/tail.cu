// The coarse tail of the V-cycle in one kernel (sm_100a): every level with at most 16 cells
// per axis — pre-smoothing residual, restriction, recursion down to the coarsest Cholesky
// solve, prolongation and post-smoothing on the way up (multigrid.py:205-222 for levels
// 0 .. LT) — runs in ONE CTA per parameter instance with all level vectors resident in
// shared memory.  Replaces 4 launches per level (coarse_kron_kernel RESID / JACOBI,
// restrict_kernel, prolong_kernel) plus coarse_solve_kernel, each latency-bound on grids this
// small, and their HBM round trips; the only global traffic is the level-LT rhs / pre-scaled
// rhs in, the level-LT correction out, and the coarsest factor.
//
// The operators are the matrix-free z-grouped Kronecker form of coarse.cu (a thread owns a
// grid column, keeps its 9G in-plane weights in registers and marches in z); every sum is
// taken in the order of the separate kernels, so the tail is bitwise the unfused path.
#include "tail.cuh"

namespace rbws {

namespace {

// T(i, i+o) of a 1D tridiagonal factor stored as [diag | upper] with stride n1 (the tables are
// staged in shared memory)
__device__ __forceinline__ double tri1(const double* f, int n1, int i, int o) {
  if (o == 0) return f[i];
  if (o > 0) return f[n1 + i];
  return f[n1 + i - 1];
}

__host__ __device__ inline int tail_vec(int n) {  // padded vector + zero tail for k = n reads
  return (n * n * n + n * n + n + 2 + 1) & ~1;
}

// in-plane weights W_g(ox, oy) of column (i, j): coarse_kron_kernel's set-up
template <int G>
__device__ void tail_weights(int n, int Q, const double* fac, const int* grp, const double* th,
                             int i, int j, bool on, double* w) {
  const int n1 = n + 1, fstride = 2 * n1;
#pragma unroll
  for (int o = 0; o < G * 9; ++o) w[o] = 0.0;
  if (!on) return;
#pragma unroll 3
  for (int t = 0; t < 3 * Q; ++t) {
    const int gt = grp[t];
    const double tq = th[t / 3];
    const double* fx = fac + ((size_t)t * 3 + 0) * fstride;
    const double* fy = fac + ((size_t)t * 3 + 1) * fstride;
    const double xv[3] = {tri1(fx, n1, i, -1), tri1(fx, n1, i, 0), tri1(fx, n1, i, 1)};
    const double yv[3] = {tq * tri1(fy, n1, j, -1), tq * tri1(fy, n1, j, 0), tq * tri1(fy, n1, j, 1)};
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (gt == g) {
#pragma unroll
        for (int oy = 0; oy < 3; ++oy)
#pragma unroll
          for (int ox = 0; ox < 3; ++ox)
            w[g * 9 + oy * 3 + ox] = fma(yv[oy], xv[ox], w[g * 9 + oy * 3 + ox]);
      }
  }
}

// z stencils of every group on planes 0 .. n: zg[k][g][3]
template <int G>
__device__ void tail_ztable(int n, int Q, const double* fac, const int* grp, double* zg) {
  const int n1 = n + 1, fstride = 2 * n1;
  for (int t = threadIdx.x; t < (n + 1) * G * 3; t += blockDim.x) {
    const int k = t / (3 * G), g = (t / 3) % G, o = t % 3 - 1;
    int rep = 0;
    for (int u = 3 * Q - 1; u >= 0; --u)
      if (grp[u] == g) rep = u;
    const double* fz = fac + ((size_t)rep * 3 + 2) * fstride;
    zg[t] = (k >= 1 && k <= n - 1) ? tri1(fz, n1, k, o) : 0.0;
  }
}

enum TailOp : int { TO_SCALE = 0, TO_RESID = 1, TO_JACOBI = 2 };

// one column of a level operation on shared-memory vectors (padded layout):
//   TO_SCALE  Y = w D^-1 B          (pre-smoothing from zero)
//   TO_RESID  Y = B - A X
//   TO_JACOBI Y = X + w D^-1 (B - A X)
template <int G, int OP>
__device__ void tail_column(int n, const double* zg, const double* w, int i, int j,
                            const double* X, const double* Bv, double* Y, double om) {
  const int n2 = n * n, hi = j * n + i;
  auto diag = [&](int k) {
    const double* zk = zg + k * G * 3;
    double dg = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) dg = fma(zk[g * 3 + 1], w[g * 9 + 4], dg);
    return dg;
  };
  if (OP == TO_SCALE) {
    double dprev = 0.0, di = 0.0;
    for (int k = 1; k < n; ++k) {
      const double dg = diag(k);
      if (dg != dprev) {
        di = 1.0 / dg;
        dprev = dg;
      }
      Y[k * n2 + hi] = om * di * Bv[k * n2 + hi];
    }
    return;
  }
  auto conv = [&](int k, double* s, double& xc) {
    const double* P = X + k * n2 + hi;
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
  double sd[G], s0[G], su[G], xd = 0.0, x0 = 0.0, xu = 0.0;
  conv(0, sd, xd);
  conv(1, s0, x0);
  double dprev = 0.0, cdi = 0.0;  // damping / diagonal, recomputed only when the diagonal changes
  for (int k = 1; k < n; ++k) {
    conv(k + 1, su, xu);
    const double* zk = zg + k * G * 3;
    double Au = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g)
      Au = fma(zk[g * 3 + 0], sd[g], fma(zk[g * 3 + 1], s0[g], fma(zk[g * 3 + 2], su[g], Au)));
    const double bv = Bv[k * n2 + hi];
    if (OP == TO_RESID) {
      Y[k * n2 + hi] = bv - Au;
    } else {
      const double dg = diag(k);
      if (dg != dprev) {
        cdi = om / dg;
        dprev = dg;
      }
      Y[k * n2 + hi] = fma(cdi, bv - Au, x0);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      sd[g] = s0[g];
      s0[g] = su[g];
    }
    x0 = xu;
  }
}

// shared-memory layout (doubles): per level l >= 1: U, R, [B (l < LT)], zg, factor tables;
// level 0: B, E; substitution vector; coarsest factor (m <= kTailLsm); theta, groups
constexpr int kTailLsm = 32;
struct TailLayout {
  int U[kTailMaxLevels + 1], R[kTailMaxLevels + 1], B[kTailMaxLevels + 1], Z[kTailMaxLevels + 1],
      F[kTailMaxLevels + 1];
  int ysub, Lsm, th, grp, total;
};
__host__ __device__ inline TailLayout tail_layout(const TailArgs& a, int G) {
  TailLayout t{};
  int p = 0;
  for (int l = a.LT; l >= 1; --l) {
    const int V = tail_vec(a.n[l]);
    t.U[l] = p; p += V;
    t.R[l] = p; p += V;
    t.B[l] = -1;
    if (l < a.LT) { t.B[l] = p; p += V; }
    t.Z[l] = p; p += ((a.n[l] + 1) * G * 3 + 1) & ~1;
    t.F[l] = p; p += a.Q * 3 * 3 * 2 * (a.n[l] + 1);
  }
  const int V0 = tail_vec(a.n[0]);
  t.B[0] = p; p += V0;
  t.R[0] = p; p += V0;
  const int m1 = a.n[0] - 1, m = m1 * m1 * m1;
  t.ysub = p; p += (m + 1) & ~1;
  t.Lsm = -1;
  if (m <= kTailLsm) { t.Lsm = p; p += m * m + (m * m & 1); }
  t.th = p; p += (a.Q + 1) & ~1;
  t.grp = p; p += (3 * a.Q + 1) / 2 * kTailMaxLevels + 2;  // ints, 3Q per level
  t.total = p;
  return t;
}

template <int G>
__global__ void __launch_bounds__(256, 2) coarse_tail_kernel(TailArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int mu = blockIdx.x;
  if (a.active && !a.active[mu]) return;
  const int tid = threadIdx.x, LT = a.LT, Q = a.Q;
  const double om = a.omega;
  const TailLayout lay = tail_layout(a, G);
  for (int t = tid; t < lay.total; t += blockDim.x) sm[t] = 0.0;
  __syncthreads();
  double* th = sm + lay.th;
  int* grps = reinterpret_cast<int*>(sm + lay.grp);  // [level - 1][3Q]
  const int n0 = a.n[0], m1 = n0 - 1, m = m1 * m1 * m1;
  {  // level-LT pre-scaled rhs, the factor tables / groups of every level, theta, the coarsest
     // factor: everything this instance reads more than once
    const int n = a.n[LT], n3 = n * n * n;
    const double* gu = a.u + (size_t)mu * n3;
    double* U = sm + lay.U[LT];
    for (int t = tid; t < n3; t += blockDim.x) U[t] = gu[t];
    for (int l = LT; l >= 1; --l) {
      const int fd = Q * 3 * 3 * 2 * (a.n[l] + 1);
      double* F = sm + lay.F[l];
      for (int t = tid; t < fd; t += blockDim.x) F[t] = __ldg(a.fac[l] + t);
      if (tid < 3 * Q) grps[(l - 1) * 3 * Q + tid] = __ldg(a.grp[l] + tid);
    }
    if (tid < Q) th[tid] = a.theta[(size_t)mu * Q + tid];
    if (lay.Lsm >= 0) {
      const double* L = a.L0 + (size_t)mu * m * m;
      for (int t = tid; t < m * m; t += blockDim.x) sm[lay.Lsm + t] = __ldg(L + t);
    }
  }
  __syncthreads();
  for (int l = LT; l >= 1; --l)
    tail_ztable<G>(a.n[l], Q, sm + lay.F[l], grps + (l - 1) * 3 * Q, sm + lay.Z[l]);
  __syncthreads();
  double w[G * 9];
  // ---- down: residual of the pre-smoothed iterate, restriction
  for (int l = LT; l >= 1; --l) {
    const int n = a.n[l];
    const int i = tid % n, j = tid / n;
    const bool col = tid < n * n, on = col && i >= 1 && j >= 1;
    double *U = sm + lay.U[l], *R = sm + lay.R[l];
    const double* zg = sm + lay.Z[l];
    // the level's rhs: the top level's stays in global memory (read by its own thread only)
    const double* Bv = l < LT ? sm + lay.B[l] : a.b + (size_t)mu * n * n * n;
    tail_weights<G>(n, Q, sm + lay.F[l], grps + (l - 1) * 3 * Q, th, i, j, on, w);
    if (l < LT) {  // u = w D^-1 b (the top level's comes from the restriction above it)
      if (on) tail_column<G, TO_SCALE>(n, zg, w, i, j, nullptr, Bv, U, om);
      __syncthreads();
    }
    if (on) tail_column<G, TO_RESID>(n, zg, w, i, j, U, Bv, R, om);
    __syncthreads();
    // B_{l-1} = P^T R_l (restrict_kernel's order of sums)
    const int nc = n / 2, nc3 = nc * nc * nc, n2 = n * n;
    const double* r = R;
    double* Bc = sm + lay.B[l - 1];
    for (int X = tid; X < nc3; X += blockDim.x) {
      const int I = X % nc, J = (X / nc) % nc, K = X / (nc * nc);
      if (I == 0 || J == 0 || K == 0) continue;
      const int c = 2 * I + n * 2 * J + n2 * 2 * K;
      double acc = 0.0;
#pragma unroll
      for (int dz = -1; dz <= 1; ++dz) {
        double pz = 0.0;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
          const int row = c + dz * n2 + dy * n;
          const double px = 0.5 * (r[row - 1] + r[row + 1]) + r[row];
          pz += (dy == 0 ? 1.0 : 0.5) * px;
        }
        acc += (dz == 0 ? 1.0 : 0.5) * pz;
      }
      Bc[X] = acc;
    }
    __syncthreads();
  }
  // ---- coarsest level: dense Cholesky solve by one warp (coarse_solve_kernel)
  if (tid < 32) {
    const int lane = tid;
    double* ysub = sm + lay.ysub;
    const double* B0 = sm + lay.B[0];
    double* E0 = sm + lay.R[0];
    auto pad = [&](int r) { return (r % m1 + 1) + n0 * ((r / m1) % m1 + 1 + n0 * (r / (m1 * m1) + 1)); };
    for (int r = lane; r < m; r += 32) ysub[r] = B0[pad(r)];
    __syncwarp();
    auto solve = [&](const double* L) {
      for (int r = 0; r < m; ++r) {  // L y = b
        double s = 0.0;
        for (int c = lane; c < r; c += 32) s = fma(L[r * m + c], ysub[c], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) ysub[r] = (ysub[r] - s) / L[r * m + r];
        __syncwarp();
      }
      for (int r = m - 1; r >= 0; --r) {  // L^T x = y
        double s = 0.0;
        for (int c = r + 1 + lane; c < m; c += 32) s = fma(L[c * m + r], ysub[c], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) ysub[r] = (ysub[r] - s) / L[r * m + r];
        __syncwarp();
      }
    };
    if (lay.Lsm >= 0) solve(sm + lay.Lsm);
    else solve(a.L0 + (size_t)mu * m * m);
    for (int r = lane; r < m; r += 32) E0[pad(r)] = ysub[r];
  }
  __syncthreads();
  // ---- up: U_l += P E_{l-1} (prolong_kernel's marching order), then the post-smoothing sweep
  for (int l = 1; l <= LT; ++l) {
    const int n = a.n[l], nc = n / 2, n2 = n * n, nc2 = nc * nc;
    const int i = tid % n, j = tid / n;
    const bool col = tid < n * n, on = col && i >= 1 && j >= 1;
    double *U = sm + lay.U[l], *R = sm + lay.R[l];
    const double* Bv = l < LT ? sm + lay.B[l] : a.b + (size_t)mu * n * n * n;
    if (on) {
      const double* e = sm + lay.R[l - 1] + (i >> 1) + nc * (j >> 1);
      const bool oi = i & 1, oj = j & 1;
      auto vxy = [&](int K) -> double {
        const double* q = e + nc2 * K;
        const double r0 = oi ? 0.5 * (q[0] + q[1]) : q[0];
        if (!oj) return r0;
        const double* q1 = q + nc;
        const double r1 = oi ? 0.5 * (q1[0] + q1[1]) : q1[0];
        return 0.5 * (r0 + r1);
      };
      int Kc = 0;
      double v0 = vxy(0), v1 = vxy(1);
      double* ucol = U + j * n + i;
      for (int k = 1; k < n; ++k) {
        const int K = k >> 1;
        if (K != Kc) {
          v0 = v1;
          v1 = vxy(K + 1);
          Kc = K;
        }
        const double pe = (k & 1) ? 0.5 * (v0 + v1) : v0;
        ucol[k * n2] = ucol[k * n2] + pe;
      }
    }
    tail_weights<G>(n, Q, sm + lay.F[l], grps + (l - 1) * 3 * Q, th, i, j, on, w);
    __syncthreads();
    if (l < LT) {
      if (on) tail_column<G, TO_JACOBI>(n, sm + lay.Z[l], w, i, j, U, Bv, R, om);
    } else if (on) {  // the level-LT correction goes straight to global memory
      tail_column<G, TO_JACOBI>(n, sm + lay.Z[l], w, i, j, U, Bv,
                                a.e + (size_t)mu * n * n * n, om);
    }
    __syncthreads();
  }
}

size_t tail_smem(const TailArgs& a, int G) {
  return (size_t)tail_layout(a, G).total * sizeof(double);
}

}  // namespace

bool coarse_tail_fits(const TailArgs& a, int G) {
  if (G < 1 || G > kCoarseMaxGroups || a.LT < 1 || a.LT > kTailMaxLevels) return false;
  for (int l = 1; l <= a.LT; ++l)
    if (a.n[l] > 16 || a.n[l] * a.n[l] > 256 || (a.n[l] & 1)) return false;
  const int m1 = a.n[0] - 1;
  if (m1 * m1 * m1 > 125) return false;
  return tail_smem(a, G) <= 227 * 1024;
}

cudaError_t coarse_tail_launch(const TailArgs& a, int G, int batch, cudaStream_t stream) {
  if (!coarse_tail_fits(a, G)) return cudaErrorInvalidValue;
  const size_t smem = tail_smem(a, G);
  const void* fn = nullptr;
  switch (G) {
    case 1: fn = (const void*)coarse_tail_kernel<1>; break;
    case 2: fn = (const void*)coarse_tail_kernel<2>; break;
    case 3: fn = (const void*)coarse_tail_kernel<3>; break;
    default: fn = (const void*)coarse_tail_kernel<4>; break;
  }
  cudaError_t e = smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  count_launch();
  switch (G) {
    case 1: coarse_tail_kernel<1><<<batch, 256, smem, stream>>>(a); break;
    case 2: coarse_tail_kernel<2><<<batch, 256, smem, stream>>>(a); break;
    case 3: coarse_tail_kernel<3><<<batch, 256, smem, stream>>>(a); break;
    default: coarse_tail_kernel<4><<<batch, 256, smem, stream>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace rbws
