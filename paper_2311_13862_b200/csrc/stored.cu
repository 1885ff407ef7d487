// Finest level of the assembled (stored-coefficient) problems: z-marching 27-point apply with
// batch-shared per-term coefficients (example-1, reference grid.py:246-255 `operator(mu) @ x`).
//
// A CTA owns TY = 256 / N full grid rows of IB parameter instances and marches through z.
// For every instance the TY rows of a plane plus one halo row above and below are ONE
// contiguous byte range of its padded vector, staged with one cp.async.bulk per
// instance into an mbarrier ring of S planes, so all 27 neighbour reads of a node are
// shared-memory reads and HBM sees every x byte once.  The per-term coefficients (the same for
// every instance of the batch: A(mu) = sum_q theta_q(mu) A_q) are read once per node and reused
// for the IB instances; instance groups are the fastest grid dimension, so the CTAs resident
// at one time work on the same tile and the coefficients come from L2.  Each term is applied
// separately (s_q = A_q x, 27 FMAs per term) and combined at the end (y = sum_q theta_q s_q):
// 27 Q + Q FP64 operations per node and instance instead of 27 (Q + 1) for combining the
// coefficients first.
#include <cstdio>
#include <cstdlib>

#include "coarse.cuh"
#include "tma.cuh"

namespace rbws {

namespace {

template <int N>
struct ZT {
  static constexpr int THREADS = 256;
  static constexpr int TY = THREADS / N;     // rows per tile (one per thread)
  static constexpr int HSZ = (TY + 2) * N;   // doubles per staged plane and instance
  // slot stride: the +x neighbour of column N-1 in the last halo row is one element past the
  // staged rows (the next row's ghost in global memory): a zeroed pad element stands in
  static constexpr int HSZP = HSZ + 2;
  static constexpr int YTILES = N / TY;
};

// forward offset o = 1..13 of the symmetric 27-point storage (coarse.cu fwd_off)
__host__ __device__ constexpr int zoff_dz(int o) { return (o - 1) < 9 ? 1 : 0; }
__host__ __device__ constexpr int zoff_dy(int o) {
  return (o - 1) < 9 ? (o - 1) / 3 - 1 : ((o - 1) < 12 ? 1 : 0);
}
__host__ __device__ constexpr int zoff_dx(int o) {
  return (o - 1) < 9 ? (o - 1) % 3 - 1 : ((o - 1) < 12 ? (o - 1) - 10 : 1);
}

#ifndef RBWS_ZM_MINB
#define RBWS_ZM_MINB 2
#endif
template <int MODE, int Q, int IB, int N, int S>
__global__ void __launch_bounds__(256, RBWS_ZM_MINB) stored_zm_kernel(const double* __restrict__ tc,
                                                        const double* __restrict__ theta,
                                                        const double* __restrict__ dinv,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ y,
                                                        const int* __restrict__ active,
                                                        double omega, int batch, int zc) {
  using G = ZT<N>;
  constexpr int TY = G::TY, HSZ = G::HSZP, YT = G::YTILES;
  constexpr int N2 = N * N, N3 = N2 * N;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);             // [S]
  double* ring = reinterpret_cast<double*>(smem + 128);          // [S][IB][HSZ]

  const int mu0 = blockIdx.x * IB;
  const int yt = blockIdx.y % YT, kc = blockIdx.y / YT;
  bool on[IB];
  int nact = 0;
#pragma unroll
  for (int u = 0; u < IB; ++u) {
    on[u] = mu0 + u < batch && (!active || active[mu0 + u]);
    nact += on[u] ? 1 : 0;
  }
  if (!nact) return;  // CTA-uniform
  const int kz = (N + zc - 1) / zc;
  const int kb = max(1, kc * kz), ke = min(N, (kc + 1) * kz);
  if (kb >= ke) return;
  const int p_first = kb - 1, p_last = ke;  // staged planes (inclusive)
  const int tid = threadIdx.x;
  const int j0 = yt * TY;
  const int i = tid % N, rl = tid / N, j = j0 + rl;
  const bool node_on = (i != 0) && (j != 0);
  const int skip = (j0 == 0) ? 1 : 0;  // row j0-1 is not needed (row 0 holds ghosts only)

  auto issue = [&](int p) {
    const int sl = (p - p_first) % S;
    const uint32_t bytes = (uint32_t)((TY + 2 - skip) * N * 8);
    mbar_arrive_expect_tx(&bar[sl], bytes * (uint32_t)nact);
    const int64_t row = (int64_t)p * N2 + (int64_t)(j0 - 1 + skip) * N;
#pragma unroll
    for (int u = 0; u < IB; ++u)
      if (on[u])
        bulk_g2s(ring + ((int64_t)sl * IB + u) * HSZ + skip * N,
                 x + (int64_t)(mu0 + u) * N3 + row, bytes, &bar[sl]);
  };
  auto wait = [&](int p) {
    const int t = p - p_first;
    mbar_wait(&bar[t % S], (uint32_t)((t / S) & 1));
  };
  if (tid < S * IB) ring[(int64_t)tid * HSZ + G::HSZ] = 0.0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);
  }
  __syncthreads();

  double th[IB][Q];
#pragma unroll
  for (int u = 0; u < IB; ++u)
#pragma unroll
    for (int q = 0; q < Q; ++q) th[u][q] = on[u] ? __ldg(theta + (int64_t)(mu0 + u) * Q + q) : 0.0;

  wait(p_first);
  wait(p_first + 1);
  int X = i + N * j + N2 * kb;  // this thread's node on plane k (global index in an instance)
  for (int k = kb; k < ke; ++k, X += N2) {
    if (k + 1 > p_first + 1) wait(k + 1);
    if (node_on) {
      const int s0 = (k - 1 - p_first) % S, s1 = (k - p_first) % S, s2 = (k + 1 - p_first) % S;
      const int c = (rl + 1) * N + i;  // centre in a staged plane
      // the per-instance vectors of the update (b, 1/diag): loads issued before the stencil
      // so their DRAM latency overlaps it
      double bv[IB], wv[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int64_t go = (int64_t)(mu0 + u) * N3 + X;
        bv[u] = (MODE != 0 && on[u]) ? __ldg(b + go) : 0.0;
        wv[u] = (MODE == 2 && dinv && on[u]) ? omega * __ldg(dinv + go) : 0.0;
      }
      double s[IB][Q];
      double cq[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) cq[q] = __ldg(tc + (int64_t)q * 14 * N3 + X);
      double xc[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        xc[u] = ring[((int64_t)s1 * IB + u) * HSZ + c];
#pragma unroll
        for (int q = 0; q < Q; ++q) s[u][q] = cq[q] * xc[u];
      }
#pragma unroll
      for (int o = 1; o < 14; ++o) {
        const int dx = zoff_dx(o), dy = zoff_dy(o), dz = zoff_dz(o);
        const int off = dx + N * (dy + N * dz);
        double cf[Q], cb[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          cf[q] = __ldg(tc + ((int64_t)q * 14 + o) * N3 + X);
          cb[q] = __ldg(tc + ((int64_t)q * 14 + o) * N3 + X - off);
        }
        const int sf = dz ? s2 : s1, sb = dz ? s0 : s1;
        const int ef = c + dx + N * dy, eb = c - dx - N * dy;
#pragma unroll
        for (int u = 0; u < IB; ++u) {
          const double xf = ring[((int64_t)sf * IB + u) * HSZ + ef];
          const double xb = ring[((int64_t)sb * IB + u) * HSZ + eb];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            s[u][q] = fma(cf[q], xf, s[u][q]);
            s[u][q] = fma(cb[q], xb, s[u][q]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        if (!on[u]) continue;
        double Au = th[u][0] * s[u][0];
#pragma unroll
        for (int q = 1; q < Q; ++q) Au = fma(th[u][q], s[u][q], Au);
        const int64_t go = (int64_t)(mu0 + u) * N3 + X;
        double out;
        if (MODE == 0) {
          out = Au;
        } else if (MODE == 1) {
          out = bv[u] - Au;
        } else if (dinv) {  // the level's 1/diag (batch setup): no per-node division
          out = fma(wv[u], bv[u] - Au, xc[u]);
        } else {
          double d = th[u][0] * cq[0];
#pragma unroll
          for (int q = 1; q < Q; ++q) d = fma(th[u][q], cq[q], d);
          out = fma(omega / d, bv[u] - Au, xc[u]);
        }
        y[go] = out;
      }
    }
    __syncthreads();  // every thread is done with plane k-1's slot
    if (tid == 0 && k - 1 + S <= p_last) issue(k - 1 + S);
  }
}

template <int MODE, int Q, int IB, int N>
cudaError_t zm_launch(const double* tc, const double* theta, const double* dinv, int batch,
                      const double* x,
                      const double* b, double* y, double omega, const LaunchCtx& lc) {
  constexpr int S = 4;
  using G = ZT<N>;
  const size_t smem = 128 + (size_t)S * IB * G::HSZP * 8;
  cudaError_t e = smem_attr((const void*)stored_zm_kernel<MODE, Q, IB, N, S>, smem);
  if (e != cudaSuccess) return e;
  const int groups = (batch + IB - 1) / IB;
  int zc = 1;  // z-chunks: at least two CTAs per SM, chunks of >= 8 planes
  while ((int64_t)groups * G::YTILES * zc < 2 * 148 && N / (zc * 2) >= 8) zc *= 2;
  dim3 grd((unsigned)groups, (unsigned)(G::YTILES * zc));
  count_launch();
  stored_zm_kernel<MODE, Q, IB, N, S><<<grd, G::THREADS, smem, lc.stream>>>(
      tc, theta, dinv, x, b, y, lc.active, omega, batch, zc);
  return cudaGetLastError();
}

template <int Q, int N>
cudaError_t zm_launch_m(int mode, const double* tc, const double* theta, const double* dinv,
                        int batch,
                        const double* x, const double* b, double* y, double omega,
                        const LaunchCtx& lc) {
  // instances per CTA: 8 for apply / residual; 4 for the Jacobi sweep, which also keeps x, b
  // and 1/diag of every instance live (8 spills at 128 registers; measured 1.96 vs 1.25 ms)
#ifndef RBWS_ZM_IB
#define RBWS_ZM_IB 8
#endif
  constexpr int IB = RBWS_ZM_IB;
  constexpr int IBJ = IB > 4 ? 4 : IB;
  switch (mode) {
    case 0: return zm_launch<0, Q, IB, N>(tc, theta, dinv, batch, x, b, y, omega, lc);
    case 1: return zm_launch<1, Q, IB, N>(tc, theta, dinv, batch, x, b, y, omega, lc);
    case 2: return zm_launch<2, Q, IBJ, N>(tc, theta, dinv, batch, x, b, y, omega, lc);
    default: return cudaErrorInvalidValue;
  }
}

template <int Q>
cudaError_t zm_launch_q(int mode, int n, const double* tc, const double* theta,
                        const double* dinv, int batch,
                        const double* x, const double* b, double* y, double omega,
                        const LaunchCtx& lc) {
  switch (n) {
    case 16: return zm_launch_m<Q, 16>(mode, tc, theta, dinv, batch, x, b, y, omega, lc);
    case 32: return zm_launch_m<Q, 32>(mode, tc, theta, dinv, batch, x, b, y, omega, lc);
    case 64: return zm_launch_m<Q, 64>(mode, tc, theta, dinv, batch, x, b, y, omega, lc);
    case 128: return zm_launch_m<Q, 128>(mode, tc, theta, dinv, batch, x, b, y, omega, lc);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool stored_zm_ok(int n, int Q, const LaunchCtx& lc) {
  static const bool on = [] {  // A/B: RBWS_FEM_ZM=0 keeps the one-node-per-thread kernel
    const char* e = getenv("RBWS_FEM_ZM");
    return !(e && atoi(e) == 0);
  }();
  if (!on || (lc.zhi > 0 && (lc.zlo != 0 || lc.zhi != n))) return false;
  return (n == 16 || n == 32 || n == 64 || n == 128) && Q >= 1 && Q <= 4;
}

cudaError_t stored_zm_launch(int mode, int n, int Q, const double* tcoef, const double* theta,
                             const double* dinv, int batch, const double* x, const double* b, double* y,
                             double omega, const LaunchCtx& lc) {
  switch (Q) {
    case 1: return zm_launch_q<1>(mode, n, tcoef, theta, dinv, batch, x, b, y, omega, lc);
    case 2: return zm_launch_q<2>(mode, n, tcoef, theta, dinv, batch, x, b, y, omega, lc);
    case 3: return zm_launch_q<3>(mode, n, tcoef, theta, dinv, batch, x, b, y, omega, lc);
    case 4: return zm_launch_q<4>(mode, n, tcoef, theta, dinv, batch, x, b, y, omega, lc);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbws
