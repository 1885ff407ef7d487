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
// exist in HBM.  Input planes (tile rows + one halo row each side) are staged
// with one TMA bulk copy per array per plane into an 8-slot mbarrier ring.
#include "coarse.cuh"
#include "tma.cuh"

namespace rbws {

constexpr int kCStages = 8;
constexpr int kCMaxPlanes = 260;  // z-factor flag table bound (planes per z-chunk + 2)

CoarseGeom coarse_geom(int n, int batch) {
  CoarseGeom g;
  int ty = 256 / n;
  if (ty < 1) ty = 1;
  if (ty > n) ty = n;
  g.ty = ty;
  g.threads = ty * n;
  g.ytiles = n / ty;
  g.zc = 1;
  while ((int64_t)g.ytiles * batch * g.zc < 2 * 148 && n / (g.zc * 2) >= 8) g.zc *= 2;
  return g;
}

struct CoarseArgs {
  int n, Q;
  CoarseGeom g;
  const double* fac;    // [Q*3][3][2][n+1]
  const double* theta;  // [batch][Q]
  const double* x;      // staged (halo)
  const double* dinv;   // staged (halo), PRE only
  const double* b;      // centre (global loads)
  double* y;
  const int* active;
  double omega;
};

enum CoarseMode : int { CM_APPLY = 0, CM_RESID = 1, CM_JACOBI = 2, CM_PRE = 3, CM_DINV = 4 };

// T(i, i+o) of a 1D tridiagonal factor stored as [diag | upper] with stride n1
__device__ __forceinline__ double tri(const double* f, int n1, int i, int o) {
  if (o == 0) return __ldg(f + i);
  if (o > 0) return __ldg(f + n1 + i);
  return __ldg(f + n1 + i - 1);
}

template <int MODE>
__global__ void __launch_bounds__(256) coarse_kernel(CoarseArgs a) {
  constexpr int NH = (MODE == CM_PRE) ? 2 : ((MODE == CM_DINV) ? 0 : 1);
  constexpr int S = kCStages;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = a.n, n1 = n + 1, Q = a.Q;
  const int ty = a.g.ty, zc = a.g.zc;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (a.active && !a.active[mu]) return;
  const int j0 = blockIdx.y * ty;
  const int tid = threadIdx.x;
  const int64_t n2 = (int64_t)n * n;
  const int64_t base = (int64_t)mu * n2 * n;
  const int kz = n / zc;
  const int kb = max(1, kc * kz), ke = min(n, (kc + 1) * kz);
  const int p_first = kb - 1, p_last = ke;
  const int np = p_last - p_first + 1;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int* zsame = reinterpret_cast<int*>(smem + 64);
  double* ring = reinterpret_cast<double*>(smem + 64 + 4 * kCMaxPlanes + 64);
  // slot = (ty+2) staged rows + 2 zero pad doubles: the 27-point corner neighbour of
  // the tile's last column/row reads one element past the staged rows (a ghost, 0)
  const int hsz = (ty + 2) * n + 2;
  auto hptr = [&](int st, int arr) { return ring + (st * NH + arr) * hsz; };

  const double* fac = a.fac;
  const int fstride = 2 * n1;  // one axis factor [diag | upper]
  auto zfac = [&](int t, int k, int oz) {  // Z factor of part t at plane k, offset oz
    return tri(fac + ((size_t)t * 3 + 2) * fstride, n1, k, oz);
  };
  if (tid == 0 && NH > 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  if (NH > 0) {  // zero the pads and (first tile) the never-staged halo row above row 0
    for (int t = tid; t < S * NH; t += blockDim.x) {
      double* sl = ring + t * hsz;
      sl[hsz - 2] = 0.0;
      sl[hsz - 1] = 0.0;
    }
    if (j0 == 0)
      for (int t = tid; t < S * NH * n; t += blockDim.x) ring[(t / n) * hsz + t % n] = 0.0;
  }
  for (int p = 1 + tid; p < np; p += blockDim.x) {
    const int k = p_first + p;
    int same = 1;
    for (int t = 0; t < 3 * Q && same; ++t)
      for (int oz = -1; oz <= 1; ++oz) same &= (zfac(t, k, oz) == zfac(t, k - 1, oz));
    zsame[p] = same;
  }
  __syncthreads();

  auto issue = [&](int p) {
    const int st = (p - p_first) & (S - 1);
    const int skip = (j0 == 0) ? 1 : 0;
    const uint32_t bytes = (uint32_t)((ty + 2 - skip) * n * 8);
    mbar_arrive_expect_tx(&bar[st], NH * bytes);
    const int64_t plane = base + (int64_t)p * n2 + (int64_t)(j0 - 1 + skip) * n;
    bulk_g2s(hptr(st, 0) + skip * n, a.x + plane, bytes, &bar[st]);
    if (NH == 2) bulk_g2s(hptr(st, 1) + skip * n, a.dinv + plane, bytes, &bar[st]);
  };
  if (NH > 0 && tid == 0)
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);

  const int i = tid % n, jl = tid / n, j = j0 + jl;
  const bool on = (i >= 1) && (j >= 1);
  const double* th = a.theta + (size_t)mu * Q;
  double c[27];  // c[(oz+1)*9 + (oy+1)*3 + (ox+1)]
  auto coeffs = [&](int k) {
#pragma unroll
    for (int o = 0; o < 27; ++o) c[o] = 0.0;
    if (!on) return;
    for (int t = 0; t < 3 * Q; ++t) {
      const double tq = th[t / 3];
      const double* fx = fac + ((size_t)t * 3 + 0) * fstride;
      const double* fy = fac + ((size_t)t * 3 + 1) * fstride;
      double X[3], Y[3], Z[3];
#pragma unroll
      for (int o = -1; o <= 1; ++o) {
        X[o + 1] = tri(fx, n1, i, o);
        Y[o + 1] = tq * tri(fy, n1, j, o);
        Z[o + 1] = zfac(t, k, o);
      }
#pragma unroll
      for (int oz = 0; oz < 3; ++oz)
#pragma unroll
        for (int oy = 0; oy < 3; ++oy) {
          const double yz = Y[oy] * Z[oz];
#pragma unroll
          for (int ox = 0; ox < 3; ++ox) c[oz * 9 + oy * 3 + ox] = fma(X[ox], yz, c[oz * 9 + oy * 3 + ox]);
        }
    }
  };

  const int hi = (jl + 1) * n + i;
  const double om = a.omega;
  if (NH > 0) {
    mbar_wait(&bar[0], 0u);
    mbar_wait(&bar[1], 0u);
  }
  for (int k = kb; k < ke; ++k) {
    const int idx = k + 1 - p_first;
    if (NH > 0) mbar_wait(&bar[idx & (S - 1)], (uint32_t)((idx / S) & 1));
    if (k == kb || !zsame[k - p_first]) coeffs(k);
    const int64_t gidx = base + (int64_t)k * n2 + (int64_t)j * n + i;
    if (MODE == CM_DINV) {
      if (on) a.y[gidx] = 1.0 / c[13];
      continue;
    }
    const int s0 = (idx - 1) & (S - 1);

    double Au = 0.0, uc = 0.0;
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      const double* X = hptr((idx - 2 + oz) & (S - 1), 0);
      const double* D = (MODE == CM_PRE) ? hptr((idx - 2 + oz) & (S - 1), 1) : nullptr;
#pragma unroll
      for (int oy = 0; oy < 3; ++oy)
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          const int id = hi + (oy - 1) * n + (ox - 1);
          const double u = (MODE == CM_PRE) ? om * D[id] * X[id] : X[id];
          Au = fma(c[oz * 9 + oy * 3 + ox], u, Au);
          if (oz == 1 && oy == 1 && ox == 1) uc = u;
        }
    }
    if (on) {
      if (MODE == CM_APPLY) a.y[gidx] = Au;
      else if (MODE == CM_RESID) a.y[gidx] = __ldg(a.b + gidx) - Au;
      else if (MODE == CM_PRE) a.y[gidx] = hptr(s0, 0)[hi] - Au;
      else a.y[gidx] = uc + om * (__ldg(a.b + gidx) - Au) / c[13];  // CM_JACOBI
    }
    if (NH > 0) {
      __syncthreads();
      if (tid == 0 && k - 1 + S <= p_last) issue(k - 1 + S);
    }
  }
}

template <int MODE>
static cudaError_t coarse_launch_m(CoarseArgs a, int batch, cudaStream_t stream) {
  constexpr int NH = (MODE == CM_PRE) ? 2 : ((MODE == CM_DINV) ? 0 : 1);
  a.g = coarse_geom(a.n, batch);
  if (a.n / a.g.zc + 2 > kCMaxPlanes) return cudaErrorInvalidValue;
  const size_t smem =
      64 + 4 * kCMaxPlanes + 64 + (size_t)kCStages * NH * ((a.g.ty + 2) * a.n + 2) * 8;
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(coarse_kernel<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  dim3 grd(1, a.g.ytiles, batch * a.g.zc);
  count_launch();
  coarse_kernel<MODE><<<grd, a.g.threads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t coarse_launch(int mode, int n, int Q, const double* fac, const double* theta,
                          int batch, const double* x, const double* b, const double* dinv,
                          double* y, double omega, const LaunchCtx& lc) {
  if (n < 2 || n > 256) return cudaErrorInvalidValue;
  CoarseArgs a{};
  a.n = n;
  a.Q = Q;
  a.fac = fac;
  a.theta = theta;
  a.x = (mode == CM_PRE) ? b : x;  // PRE stages the right-hand side (u = w dinv b)
  a.b = b;
  a.dinv = dinv;
  a.y = y;
  a.active = lc.active;
  a.omega = omega;
  switch (mode) {
    case CM_APPLY: return coarse_launch_m<CM_APPLY>(a, batch, lc.stream);
    case CM_RESID: return coarse_launch_m<CM_RESID>(a, batch, lc.stream);
    case CM_JACOBI: return coarse_launch_m<CM_JACOBI>(a, batch, lc.stream);
    case CM_PRE: return coarse_launch_m<CM_PRE>(a, batch, lc.stream);
    case CM_DINV: return coarse_launch_m<CM_DINV>(a, batch, lc.stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbws

namespace rbws {

// ---------------------------------------------------------------- coarsest level
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
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < m; ++c) {  // right-looking Cholesky, lower triangle
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
  double* L = Lout + (int64_t)mu * m * m;
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
    const int r = t / m, s = t % m;
    L[t] = (s <= r) ? A[t] : 0.0;
  }
  if (threadIdx.x == 0 && status) status[mu] = bad;
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
