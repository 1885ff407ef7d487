// L1ROC reduced-model kernels (reference rb.py): sampled term projections,
// batched online least squares with the L1 indicator, warm-start expansion,
// DEIM residual/argmax and a small dense solver.
#include <cfloat>

#include "l1roc.cuh"

namespace rbws {

// ---------------------------------------------------------------- projections
// Bq[q][m][c] = (A_q w_c)(rows[m]) with the separable term-q 7-point stencil
__global__ void l1roc_project_kernel(int n, int Q, const double* __restrict__ face,
                                     const double* __restrict__ node,
                                     const double* __restrict__ W, int64_t Wstride, int N,
                                     const int64_t* __restrict__ rows, int M,
                                     double* __restrict__ Bq) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)Q * M * N) return;
  const int c = t % N, m = (t / N) % M, q = t / ((int64_t)N * M);
  const int64_t X = rows[m];
  const int i = X % n, j = (X / n) % n, k = X / ((int64_t)n * n);
  const int n1 = n + 1;
  const double* w = W + (int64_t)c * Wstride;
  const double* F = face + (size_t)q * 3 * n;
  const double* Nd = node + (size_t)q * 9 * n1;
  const int xyz[3] = {i, j, k};
  const int64_t stride[3] = {1, n, (int64_t)n * n};
  const double wc = w[X];
  double acc = 0.0;
  for (int d = 0; d < 3; ++d) {
    double lat = 1.0;
    for (int a = 0; a < 3; ++a)
      if (a != d) lat *= Nd[((d * 3) + a) * n1 + xyz[a]];
    const double wp = F[d * n + xyz[d]] * lat, wm = F[d * n + xyz[d] - 1] * lat;
    acc += wp * (wc - w[X + stride[d]]) + wm * (wc - w[X - stride[d]]);
  }
  Bq[t] = acc;
}

cudaError_t l1roc_project(int n, int Q, const double* face, const double* node, const double* W,
                          int64_t Wstride, int N, const int64_t* rows, int M, double* Bq,
                          cudaStream_t stream) {
  const int64_t tot = (int64_t)Q * M * N;
  if (tot == 0) return cudaSuccess;
  count_launch();
  l1roc_project_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, stream>>>(n, Q, face, node, W,
                                                                          Wstride, N, rows, M, Bq);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- online LS
__device__ __forceinline__ bool warp_id_is_zero() { return (threadIdx.x >> 5) == 0; }

// one block per instance; Householder QR of the M x N sampled matrix in smem
__global__ void __launch_bounds__(128) l1roc_online_kernel(int M, int N, int Q,
                                                           const double* __restrict__ theta,
                                                           const double* __restrict__ Bq,
                                                           const double* __restrict__ bs,
                                                           int64_t bs_stride,
                                                           const double* __restrict__ T,
                                                           double* __restrict__ a_out,
                                                           double* __restrict__ c_out,
                                                           double* __restrict__ ind,
                                                           int* __restrict__ status) {
  extern __shared__ double sm[];
  double* B = sm;               // column-major [N][M]
  double* rhs = B + M * N;      // [M]
  double* red = rhs + M;        // [32]
  double* sol = red + 32;       // [N]
  double* Rw = sol + N;         // [N][N] scratch: R^-1 (rank certificate) / Jacobi SVD
  __shared__ int s_bad;
  __shared__ double s_cert[2];
  const int mu = blockIdx.x;
  const int tid = threadIdx.x;
  const double* th = theta + (int64_t)mu * Q;
  for (int t = tid; t < M * N; t += blockDim.x) {
    const int m = t / N, c = t % N;
    double v = 0.0;
    for (int q = 0; q < Q; ++q) v = fma(th[q], Bq[((int64_t)q * M + m) * N + c], v);
    B[c * M + m] = v;
  }
  for (int m = tid; m < M; m += blockDim.x) rhs[m] = bs[mu * bs_stride + m];
  __syncthreads();
  int bad = 0;
  for (int j = 0; j < N; ++j) {
    double* col = B + j * M;
    double part = 0.0;
    for (int m = j + tid; m < M; m += blockDim.x) part = fma(col[m], col[m], part);
    const double nrm2 = block_reduce_sum(part, red);
    __syncthreads();
    if (tid == 0) red[0] = nrm2;
    __syncthreads();
    const double nrm = sqrt(red[0]);
    const double x0 = col[j];
    const double alpha = (x0 >= 0.0) ? -nrm : nrm;  // R_jj
    // v = x - alpha e_j (stored in col[j..]), tau = 1/(alpha (alpha - x0)) * ... use v^T v
    __syncthreads();
    if (nrm == 0.0) {
      if (tid == 0) col[j] = 0.0;
      __syncthreads();
      continue;
    }
    if (tid == 0) col[j] = x0 - alpha;
    __syncthreads();
    const double vtv = 2.0 * nrm * (nrm + fabs(x0));  // ||x - alpha e_j||^2
    // apply H = I - 2 v v^T / vtv to remaining columns and rhs
    for (int c = j + 1; c <= N; ++c) {
      double* y = (c < N) ? B + c * M : rhs;
      double pd = 0.0;
      for (int m = j + tid; m < M; m += blockDim.x) pd = fma(col[m], y[m], pd);
      const double s = block_reduce_sum(pd, red);
      __syncthreads();
      if (tid == 0) red[0] = s;
      __syncthreads();
      const double f = 2.0 * red[0] / vtv;
      for (int m = j + tid; m < M; m += blockDim.x) y[m] = fma(-f, col[m], y[m]);
      __syncthreads();
    }
    if (tid == 0) col[j] = alpha;  // R_jj (below-diagonal part of v no longer needed)
    __syncthreads();
  }
  // ---- rank test with numpy's lstsq rule (rb.py:174-179: SVD, rcond = eps max(M, N),
  // rank = #{s_i > rcond s_max}).  Certificate first: s_max <= ||R||_F and
  // s_min >= 1 / ||R^-1||_F, so 1/||R^-1||_F > rcond ||R||_F proves full rank; otherwise the
  // singular values of R are computed (one-sided Jacobi, warp 0) and counted.
  const double rcond = DBL_EPSILON * (double)(M > N ? M : N);
  {
    double fr = 0.0;
    int zero = 0;
    for (int t = tid; t < N * N; t += blockDim.x) {
      const int r = t % N, c = t / N;
      const double v = (r <= c) ? B[c * M + r] : 0.0;
      fr = fma(v, v, fr);
      if (r == c && v == 0.0) zero = 1;
    }
    const double frs = block_reduce_sum(fr, red);
    if (tid == 0) {
      s_cert[0] = frs;
      s_bad = 0;
    }
    __syncthreads();
    if (zero) s_bad = 2;  // exactly singular R: s_min = 0
    __syncthreads();
    // ||R^-1||_F^2: column k of R^-1 by back substitution (one thread per column)
    double inv2 = 0.0;
    if (s_bad == 0) {
      for (int k = tid; k < N; k += blockDim.x) {
        double* x = Rw + k * N;
        for (int r = N - 1; r >= 0; --r) {
          double v = (r == k) ? 1.0 : 0.0;
          if (r <= k)
            for (int c = r + 1; c <= k; ++c) v -= B[c * M + r] * x[c];
          x[r] = (r <= k) ? v / B[r * M + r] : 0.0;
          inv2 = fma(x[r], x[r], inv2);
        }
      }
    }
    const double inv2s = block_reduce_sum(inv2, red);
    if (tid == 0) s_cert[1] = inv2s;
    __syncthreads();
    const bool certain = s_bad == 0 && 1.0 / sqrt(s_cert[1]) > rcond * sqrt(s_cert[0]);
    if (!certain && warp_id_is_zero()) {
      // one-sided Jacobi on the columns of R (lanes over rows), cyclic pair order
      const int lane = tid & 31;
      for (int t = lane; t < N * N; t += 32) {
        const int r = t % N, c = t / N;
        Rw[c * N + r] = (r <= c) ? B[c * M + r] : 0.0;
      }
      __syncwarp();
      for (int sweep = 0; sweep < 40; ++sweep) {
        int rotated = 0;
        for (int p = 0; p < N - 1; ++p)
          for (int q = p + 1; q < N; ++q) {
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int r = lane; r < N; r += 32) {
              const double xp = Rw[p * N + r], xq = Rw[q * N + r];
              al = fma(xp, xp, al);
              be = fma(xq, xq, be);
              ga = fma(xp, xq, ga);
            }
            for (int o = 16; o > 0; o >>= 1) {
              al += __shfl_xor_sync(0xffffffffu, al, o);
              be += __shfl_xor_sync(0xffffffffu, be, o);
              ga += __shfl_xor_sync(0xffffffffu, ga, o);
            }
            if (fabs(ga) <= DBL_EPSILON * sqrt(al * be) || ga == 0.0) continue;
            rotated = 1;
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
            for (int r = lane; r < N; r += 32) {
              const double xp = Rw[p * N + r], xq = Rw[q * N + r];
              Rw[p * N + r] = cs * xp - sn * xq;
              Rw[q * N + r] = sn * xp + cs * xq;
            }
            __syncwarp();
          }
        if (!rotated) break;
      }
      // singular values = column norms
      double smax = 0.0;
      for (int c = 0; c < N; ++c) {
        double v = 0.0;
        for (int r = lane; r < N; r += 32) v = fma(Rw[c * N + r], Rw[c * N + r], v);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        smax = fmax(smax, sqrt(v));
        if (lane == 0) sol[c] = sqrt(v);
      }
      __syncwarp();
      if (lane == 0) {
        int rank = 0;
        for (int c = 0; c < N; ++c) rank += sol[c] > rcond * smax ? 1 : 0;
        s_bad = rank < N ? 1 : 0;
      }
    }
    __syncthreads();
    bad = s_bad != 0;
  }
  if (tid == 0) {
    // back substitution R a = (Q^T b)[0:N]
    for (int j = N - 1; j >= 0; --j) {
      double s = rhs[j];
      for (int c = j + 1; c < N; ++c) s -= B[c * M + j] * sol[c];
      sol[j] = bad ? 0.0 : s / B[j * M + j];
    }
    double* ao = a_out + (int64_t)mu * N;
    for (int j = 0; j < N; ++j) ao[j] = sol[j];
    if (T) {
      // snapshot coordinates c = T^{-1} a (T upper triangular, row-major)
      double l1 = 0.0;
      double* co = c_out + (int64_t)mu * N;
      for (int j = N - 1; j >= 0; --j) {
        double s = sol[j];
        for (int c = j + 1; c < N; ++c) s -= T[j * N + c] * co[c];
        co[j] = s / T[j * N + j];
      }
      for (int j = 0; j < N; ++j) l1 += fabs(co[j]);
      ind[mu] = l1;
    }
    status[mu] = bad;
  }
}

cudaError_t l1roc_online(int count, int Q, int M, int N, const double* theta, const double* Bq,
                         const double* bs, int64_t bs_stride, const double* T, double* a,
                         double* c, double* ind, int* status, cudaStream_t stream) {
  const size_t smem = sizeof(double) * ((size_t)M * N + M + 32 + N + (size_t)N * N);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(l1roc_online_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  l1roc_online_kernel<<<count, 128, smem, stream>>>(M, N, Q, theta, Bq, bs, bs_stride, T, a, c,
                                                     ind, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- expansion
// x[mu] = W a[mu].  A thread holds its node's N basis values in registers
// (NB >= N, zero padded) and sweeps a chunk of instances whose coefficient
// vectors sit in shared memory (broadcast reads), so W is read once per chunk
// and each output costs N FMAs + N/2 128-bit shared loads.
template <int NB>
struct ExpandChunk {
  static constexpr int value = NB <= 16 ? 256 : (NB <= 32 ? 128 : 64);  // <= 32 KB of smem
};

template <int NB>
__global__ void __launch_bounds__(256) expand_kernel(int64_t n3, const double* __restrict__ W,
                                                     int64_t Wstride, int N,
                                                     const double* __restrict__ a, int count,
                                                     double* __restrict__ x) {
  constexpr int kExpandChunk = ExpandChunk<NB>::value;
  __shared__ __align__(16) double as[kExpandChunk * NB];
  const int m0 = blockIdx.y * kExpandChunk;
  const int m1 = min(count, m0 + kExpandChunk);
  for (int t = threadIdx.x; t < kExpandChunk * NB; t += blockDim.x) {
    const int mu = m0 + t / NB, c = t % NB;
    as[t] = (mu < m1 && c < N) ? a[(int64_t)mu * N + c] : 0.0;
  }
  __syncthreads();
  const int64_t X = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (X >= n3) return;
  double w[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) w[c] = (c < N) ? __ldg(W + c * Wstride + X) : 0.0;
  // four instances per trip: independent FMA chains and stores in flight
#pragma unroll 4
  for (int mu = m0; mu < m1; ++mu) {
    const double2* am = reinterpret_cast<const double2*>(as + (mu - m0) * NB);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int c = 0; c < NB / 2; ++c) {
      const double2 v = am[c];
      s0 = fma(w[2 * c], v.x, s0);
      s1 = fma(w[2 * c + 1], v.y, s1);
    }
    x[(int64_t)mu * n3 + X] = s0 + s1;
  }
}

template <int NB>
static cudaError_t expand_nb(int64_t n3, int count, const double* W, int64_t Wstride, int N,
                            const double* a, double* x, cudaStream_t stream) {
  constexpr int ch = ExpandChunk<NB>::value;
  dim3 grd((unsigned)((n3 + 255) / 256), (count + ch - 1) / ch);
  count_launch();
  expand_kernel<NB><<<grd, 256, 0, stream>>>(n3, W, Wstride, N, a, count, x);
  return cudaGetLastError();
}

cudaError_t expand(int n, int count, const double* W, int64_t Wstride, int N, const double* a,
                   double* x, cudaStream_t stream) {
  const int64_t n3 = (int64_t)n * n * n;
  if (N <= 8) return expand_nb<8>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 16) return expand_nb<16>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 20) return expand_nb<20>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 24) return expand_nb<24>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 32) return expand_nb<32>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 48) return expand_nb<48>(n3, count, W, Wstride, N, a, x, stream);
  if (N <= 64) return expand_nb<64>(n3, count, W, Wstride, N, a, x, stream);
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- basis projection
// out[m][a] = sum_x W[a][x] v[m][x]: the W^T v of the multispace preconditioner's Galerkin
// correction (reference msrb.py:53-85, rb.py:71-83).  Tall-skinny and memory-bound: a CTA
// takes a chunk of x for IB instances and NB basis vectors (IB x NB accumulators per
// thread); instance groups are the fastest grid dimension, so the basis chunk is an L2 hit
// for every group after the first and HBM sees v and W once.  Per-CTA sums go to fixed
// slots and are added in a fixed order (deterministic).
#ifndef RBWS_DOT_EPT
#define RBWS_DOT_EPT 32
#endif
constexpr int kDotIB = 4, kDotNB = 8, kDotEPT = RBWS_DOT_EPT;
__global__ void __launch_bounds__(256) basis_dot_kernel(int64_t n3, int count,
                                                        const double* __restrict__ W,
                                                        int64_t Wstride, int N,
                                                        const double* __restrict__ v,
                                                        int64_t vstride,
                                                        double* __restrict__ part) {
  const int m0 = blockIdx.x * kDotIB, xc = blockIdx.y, a0 = blockIdx.z * kDotNB;
  const int64_t x0 = (int64_t)xc * 256 * kDotEPT;
  double acc[kDotIB][kDotNB];
#pragma unroll
  for (int u = 0; u < kDotIB; ++u)
#pragma unroll
    for (int a = 0; a < kDotNB; ++a) acc[u][a] = 0.0;
#pragma unroll
  for (int e = 0; e < kDotEPT; ++e) {
    const int64_t x = x0 + e * 256 + threadIdx.x;
    if (x >= n3) break;
    double wv[kDotNB], vv[kDotIB];
#pragma unroll
    for (int a = 0; a < kDotNB; ++a) wv[a] = (a0 + a < N) ? __ldg(W + (int64_t)(a0 + a) * Wstride + x) : 0.0;
#pragma unroll
    for (int u = 0; u < kDotIB; ++u) vv[u] = (m0 + u < count) ? __ldg(v + (int64_t)(m0 + u) * vstride + x) : 0.0;
#pragma unroll
    for (int u = 0; u < kDotIB; ++u)
#pragma unroll
      for (int a = 0; a < kDotNB; ++a) acc[u][a] = fma(wv[a], vv[u], acc[u][a]);
  }
  __shared__ double red[8][kDotIB * kDotNB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < kDotIB; ++u)
#pragma unroll
    for (int a = 0; a < kDotNB; ++a) {
      double s = acc[u][a];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp][u * kDotNB + a] = s;
    }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < kDotIB * kDotNB) {
    double s = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) s += red[w8][t];
    const int u = t / kDotNB, a = t % kDotNB;
    if (m0 + u < count && a0 + a < N)
      part[((int64_t)(m0 + u) * N + a0 + a) * gridDim.y + xc] = s;
  }
}

__global__ void basis_dot_final_kernel(int total, int nchunks, const double* __restrict__ part,
                                       double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[(int64_t)t * nchunks + c];
  out[t] = s;
}

size_t basis_dot_scratch(int64_t n3, int count, int N) {
  const int64_t chunks = (n3 + 256 * kDotEPT - 1) / (256 * kDotEPT);
  return (size_t)count * N * chunks * sizeof(double);
}

cudaError_t basis_dot(int64_t n3, int count, const double* W, int64_t Wstride, int N,
                      const double* v, int64_t vstride, double* out, double* scratch,
                      cudaStream_t stream) {
  const int64_t chunks = (n3 + 256 * kDotEPT - 1) / (256 * kDotEPT);
  dim3 grd((unsigned)((count + kDotIB - 1) / kDotIB), (unsigned)chunks,
           (unsigned)((N + kDotNB - 1) / kDotNB));
  count_launch();
  basis_dot_kernel<<<grd, 256, 0, stream>>>(n3, count, W, Wstride, N, v, vstride, scratch);
  const int total = count * N;
  count_launch();
  basis_dot_final_kernel<<<(total + 127) / 128, 128, 0, stream>>>(total, (int)chunks, scratch, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- DEIM step
struct ArgMax {
  double v;
  int64_t i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  // larger value wins; ties -> smaller index (np.argmax first occurrence)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__global__ void __launch_bounds__(256) deim_rho_kernel(int n, int ghosts,
                                                       const double* __restrict__ W,
                                                       int64_t Wstride, int N,
                                                       const double* __restrict__ c,
                                                       const double* __restrict__ v,
                                                       const uint8_t* __restrict__ excl,
                                                       double* __restrict__ rho,
                                                       ArgMax* __restrict__ part_arg,
                                                       double* __restrict__ part_max) {
  __shared__ ArgMax sa[256];
  __shared__ double sv[256], sr[256];
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t X = (int64_t)blockIdx.x * 256 + threadIdx.x;
  ArgMax best{-1.0, INT64_MAX};
  double mv = 0.0, mr = 0.0;
  if (X < n3) {
    const int i = X % n, j = (X / n) % n, k = X / ((int64_t)n * n);
    double r = v[X];
    for (int q = 0; q < N; ++q) r -= W[q * Wstride + X] * c[q];
    // padded layout: entries with a zero coordinate are ghosts; full-node layout (ghosts = 0):
    // every node is admissible (Dirichlet nodes hold zeros, free x = 1 face edges included)
    const bool interior = !ghosts || (i && j && k);
    if (!interior) r = 0.0;
    rho[X] = r;
    if (interior) {
      mv = fabs(v[X]);
      mr = fabs(r);
      if (!(excl && excl[X])) best = ArgMax{fabs(r), X};
    }
  }
  sa[threadIdx.x] = best;
  sv[threadIdx.x] = mv;
  sr[threadIdx.x] = mr;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] = better(sa[threadIdx.x], sa[threadIdx.x + s]);
      sv[threadIdx.x] = fmax(sv[threadIdx.x], sv[threadIdx.x + s]);
      sr[threadIdx.x] = fmax(sr[threadIdx.x], sr[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_arg[blockIdx.x] = sa[0];
    part_max[2 * blockIdx.x] = sv[0];
    part_max[2 * blockIdx.x + 1] = sr[0];
  }
}

__global__ void deim_final_kernel(int nblocks, const ArgMax* __restrict__ part_arg,
                                  const double* __restrict__ part_max,
                                  const double* __restrict__ rho, int64_t* out_idx,
                                  double* out_vals) {
  __shared__ ArgMax sa[256];
  __shared__ double sv[256], sr[256];
  ArgMax best{-1.0, INT64_MAX};
  double mv = 0.0, mr = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) {
    best = better(best, part_arg[b]);
    mv = fmax(mv, part_max[2 * b]);
    mr = fmax(mr, part_max[2 * b + 1]);
  }
  sa[threadIdx.x] = best;
  sv[threadIdx.x] = mv;
  sr[threadIdx.x] = mr;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] = better(sa[threadIdx.x], sa[threadIdx.x + s]);
      sv[threadIdx.x] = fmax(sv[threadIdx.x], sv[threadIdx.x + s]);
      sr[threadIdx.x] = fmax(sr[threadIdx.x], sr[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t idx = sa[0].i;
    out_idx[0] = (sa[0].v >= 0.0) ? idx : -1;
    out_vals[0] = (sa[0].v >= 0.0) ? rho[idx] : 0.0;  // pivot
    out_vals[1] = sv[0];                              // max |v|
    out_vals[2] = sr[0];                              // max |rho|
  }
}

__global__ void __launch_bounds__(256) scale_kernel(int64_t n3, double* __restrict__ col,
                                                    const double* __restrict__ vals) {
  const int64_t X = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const double piv = vals[0];
  if (X < n3 && piv != 0.0) col[X] = col[X] / piv;
}

cudaError_t deim_step(int n, const double* W, int64_t Wstride, int N, const double* c,
                      const double* v, const uint8_t* excl, double* col, int64_t* out_idx,
                      double* out_vals, void* scratch, cudaStream_t stream, bool ghosts) {
  const int64_t n3 = (int64_t)n * n * n;
  const int nb = (int)((n3 + 255) / 256);
  ArgMax* pa = (ArgMax*)scratch;
  double* pm = (double*)(pa + nb);
  count_launch();
  deim_rho_kernel<<<nb, 256, 0, stream>>>(n, ghosts ? 1 : 0, W, Wstride, N, c, v, excl, col,
                                          pa, pm);
  count_launch();
  deim_final_kernel<<<1, 256, 0, stream>>>(nb, pa, pm, col, out_idx, out_vals);
  count_launch();
  scale_kernel<<<nb, 256, 0, stream>>>(n3, col, out_vals);
  return cudaGetLastError();
}

size_t deim_scratch_bytes(int n) {
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t nb = (n3 + 255) / 256;
  return nb * (sizeof(ArgMax) + 2 * sizeof(double)) + 64;
}

// ---------------------------------------------------------------- dense solve
__global__ void dense_solve_kernel(int m, const double* __restrict__ Ain,
                                   const double* __restrict__ bin, double* __restrict__ x,
                                   int* status) {
  extern __shared__ double A[];  // [m][m+1]
  const int w = m + 1;
  for (int t = threadIdx.x; t < m * m; t += blockDim.x) A[(t / m) * w + t % m] = Ain[t];
  for (int t = threadIdx.x; t < m; t += blockDim.x) A[t * w + m] = bin[t];
  __shared__ int piv;
  __shared__ int sing;
  if (threadIdx.x == 0) sing = 0;
  __syncthreads();
  for (int c = 0; c < m; ++c) {
    if (threadIdx.x == 0) {
      int p = c;
      double best = fabs(A[c * w + c]);
      for (int r = c + 1; r < m; ++r)
        if (fabs(A[r * w + c]) > best) { best = fabs(A[r * w + c]); p = r; }
      piv = p;
      if (best == 0.0) sing = 1;
    }
    __syncthreads();
    if (piv != c)
      for (int t = threadIdx.x; t <= m; t += blockDim.x) {
        const double tmp = A[c * w + t];
        A[c * w + t] = A[piv * w + t];
        A[piv * w + t] = tmp;
      }
    __syncthreads();
    const double d = A[c * w + c];
    for (int r = c + 1 + threadIdx.x; r < m; r += blockDim.x) {
      const double f = (d != 0.0) ? A[r * w + c] / d : 0.0;
      for (int t = c; t <= m; ++t) A[r * w + t] -= f * A[c * w + t];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int r = m - 1; r >= 0; --r) {
      double s = A[r * w + m];
      for (int t = r + 1; t < m; ++t) s -= A[r * w + t] * x[t];
      x[r] = (A[r * w + r] != 0.0) ? s / A[r * w + r] : 0.0;
    }
    if (status) status[0] = sing;
  }
}

cudaError_t dense_solve(int m, const double* A, const double* b, double* x, int* status,
                        cudaStream_t stream) {
  const size_t smem = sizeof(double) * (size_t)m * (m + 1);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(dense_solve_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  dense_solve_kernel<<<1, 128, smem, stream>>>(m, A, b, x, status);
  return cudaGetLastError();
}

}  // namespace rbws
