// Batched lexicographic Gauss-Seidel sweeps (reference smoother="gs": forward sweeps before
// and backward sweeps after the coarse-grid correction, multigrid.py:132-152; the sweep is
// _smoothers.pyx:14-28 csr_gauss_seidel).
//
// A lexicographic sweep updates node X from the new values of its lower-index neighbours
// and the old values of its upper ones.  Nodes on one hyperplane are independent and a
// hyperplane depends only on earlier ones: for the 7-point finest stencil the planes
// i + j + k = w, for the 27-point coarse stencils i + 2j + 4k = w (every neighbour offset
// changes w by a non-zero amount, lower neighbours by a negative one).  One CTA per
// instance walks the hyperplanes in order with a barrier between them, so the result is
// the sequential sweep's.  Each row sums its off-diagonal terms in the reference's CSR
// order (ascending column index) with separately rounded multiply and add, as the
// compiled loop does (`rsum += data[jj] * x[indices[jj]]`); Dirichlet ghost neighbours,
// absent from the reference's rows, hold 0 and add exactly 0.
//
// Access is scattered (one node per grid row per hyperplane), so a sweep is bound by
// latency and L2, not HBM: it is the parity path for smoother="gs", not a fast path (the
// reference's default for these isotropic problems is damped Jacobi).
#include "gs.cuh"

namespace rbws {

template <bool FWD>
__global__ void __launch_bounds__(512) gs7_kernel(int n, const double* __restrict__ wface,
                                                  int64_t ws, const double* __restrict__ bb,
                                                  double* xx, const int* __restrict__ active) {
  const int mu = blockIdx.x;
  if (active && !active[mu]) return;
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n, base = (int64_t)mu * n3;
  const double* WX = wface + base;
  const double* WY = wface + ws + base;
  const double* WZ = wface + 2 * ws + base;
  const double* b = bb + base;
  double* x = xx + base;
  const int m = n - 1;
  const int wlo = 3, whi = 3 * m;
  for (int s = 0; s <= whi - wlo; ++s) {
    const int w = FWD ? wlo + s : whi - s;
    const int klo = max(1, w - 2 * m), khi = min(m, w - 2);
    const int cnt = (khi - klo + 1) * m;
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int k = klo + t / m, j = 1 + t % m, i = w - j - k;
      if (i < 1 || i > m) continue;
      const int64_t X = i + (int64_t)n * (j + (int64_t)n * k);
      const double wzm = WZ[X - n2], wym = WY[X - n], wxm = WX[X - 1];
      const double wxp = WX[X], wyp = WY[X], wzp = WZ[X];
      // CSR order: (k-1), (j-1), (i-1), (i+1), (j+1), (k+1); entries -w
      double rs = __dmul_rn(-wzm, x[X - n2]);
      rs = __dadd_rn(rs, __dmul_rn(-wym, x[X - n]));
      rs = __dadd_rn(rs, __dmul_rn(-wxm, x[X - 1]));
      rs = __dadd_rn(rs, __dmul_rn(-wxp, x[X + 1]));
      rs = __dadd_rn(rs, __dmul_rn(-wyp, x[X + n]));
      rs = __dadd_rn(rs, __dmul_rn(-wzp, x[X + n2]));
      const double d = ((wxp + wxm) + (wyp + wym)) + (wzp + wzm);
      x[X] = __ddiv_rn(__dsub_rn(b[X], rs), d);
    }
    __syncthreads();  // hyperplane w complete (global writes visible to the block)
  }
}

// forward offsets o = 1..13 (dz, dy, dx): dz=+1 rows (o 1..9), dz=0 dy=+1 (10..12), dx=+1 (13)
__device__ __forceinline__ int64_t off27(int o, int64_t n) {
  const int t = o - 1;
  int dx, dy, dz;
  if (t < 9) { dz = 1; dy = t / 3 - 1; dx = t % 3 - 1; }
  else if (t < 12) { dz = 0; dy = 1; dx = t - 10; }
  else { dz = 0; dy = 0; dx = 1; }
  return dx + n * (dy + n * dz);
}

template <bool FWD>
__global__ void __launch_bounds__(512) gs27_kernel(int n, const double* __restrict__ coef,
                                                   const double* __restrict__ bb, double* xx,
                                                   const int* __restrict__ active) {
  const int mu = blockIdx.x;
  if (active && !active[mu]) return;
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n, base = (int64_t)mu * n3;
  const double* C = coef + (int64_t)mu * 14 * n3;
  const double* b = bb + base;
  double* x = xx + base;
  const int m = n - 1;
  const int wlo = 7, whi = 7 * m;
  // CSR order of a row: negative offsets ascending (-o for o = 9..1, 12, 11, 10, 13),
  // then positive ones ascending (o = 13, 10, 11, 12, 1..9)
  constexpr int neg[13] = {9, 8, 7, 6, 5, 4, 3, 2, 1, 12, 11, 10, 13};
  constexpr int pos[13] = {13, 10, 11, 12, 1, 2, 3, 4, 5, 6, 7, 8, 9};
  for (int s = 0; s <= whi - wlo; ++s) {
    const int w = FWD ? wlo + s : whi - s;
    // i + 2j in [3, 3m]  ->  k in [ceil((w - 3m)/4), floor((w - 3)/4)]
    const int klo = max(1, (w - 3 * m + 3) / 4), khi = min(m, (w - 3) / 4);
    const int cnt = (khi - klo + 1) * m;
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int k = klo + t / m, j = 1 + t % m, i = w - 2 * j - 4 * k;
      if (i < 1 || i > m) continue;
      const int64_t X = i + (int64_t)n * (j + (int64_t)n * k);
      double rs = 0.0;
#pragma unroll
      for (int q = 0; q < 13; ++q) {
        const int64_t o = off27(neg[q], n);
        rs = __dadd_rn(rs, __dmul_rn(C[neg[q] * n3 + X - o], x[X - o]));
      }
#pragma unroll
      for (int q = 0; q < 13; ++q) {
        const int64_t o = off27(pos[q], n);
        rs = __dadd_rn(rs, __dmul_rn(C[pos[q] * n3 + X], x[X + o]));
      }
      x[X] = __ddiv_rn(__dsub_rn(b[X], rs), C[X]);
    }
    __syncthreads();
  }
}

cudaError_t gs7_sweep(int n, int batch, const double* wface, int64_t wstride, const double* b,
                      double* x, bool forward, const LaunchCtx& lc) {
  if (!wface) return cudaErrorInvalidValue;
  count_launch();
  if (forward) gs7_kernel<true><<<batch, 512, 0, lc.stream>>>(n, wface, wstride, b, x, lc.active);
  else gs7_kernel<false><<<batch, 512, 0, lc.stream>>>(n, wface, wstride, b, x, lc.active);
  return cudaGetLastError();
}

cudaError_t gs27_sweep(int n, int batch, const double* coef, const double* b, double* x,
                       bool forward, const LaunchCtx& lc) {
  if (!coef) return cudaErrorInvalidValue;
  count_launch();
  if (forward) gs27_kernel<true><<<batch, 512, 0, lc.stream>>>(n, coef, b, x, lc.active);
  else gs27_kernel<false><<<batch, 512, 0, lc.stream>>>(n, coef, b, x, lc.active);
  return cudaGetLastError();
}

}  // namespace rbws
