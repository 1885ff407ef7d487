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

namespace rbws {
namespace {

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

// lower band of the plane blocks (planar = 1: systems = instances x planes, M = (c+1)^2,
// w = c+2) or of the whole level (planar = 0: M = (c+1)^3, w = (c+1)^2 + c + 2):
// band[(s*M + r)*(w+1) + d] = A[r, r-d]; Dirichlet rows -> identity rows
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
  double* row = band + (s * M + r) * (w + 1);
  for (int d = 0; d <= w; ++d) row[d] = 0.0;
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
// (w x w) triangle updated in parallel); info[s] = 0 or the first non-positive pivot + 1
__global__ void band_factor_kernel(int64_t nsys, int64_t M, int w, double* __restrict__ band,
                                   int* __restrict__ info) {
  const int64_t s = blockIdx.x;
  if (s >= nsys) return;
  double* B = band + s * M * (w + 1);
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t j = 0; j < M; ++j) {
    if (threadIdx.x == 0) {
      const double a = B[j * (w + 1)];
      if (!(a > 0.0) && !bad) bad = (int)(j + 1);
      piv = a > 0.0 ? sqrt(a) : 1.0;
      B[j * (w + 1)] = piv;
    }
    __syncthreads();
    const double p = piv;
    for (int t = 1 + threadIdx.x; t <= w; t += blockDim.x)
      if (j + t < M) B[(j + t) * (w + 1) + t] /= p;
    __syncthreads();
    // A[j+a][j+b] -= L[j+a][j] L[j+b][j], 1 <= b <= a <= w
    for (int a = 1 + warp; a <= w; a += nw) {
      if (j + a >= M) break;
      const double la = B[(j + a) * (w + 1) + a];
      for (int bb = 1 + lane; bb <= a; bb += 32)
        B[(j + a) * (w + 1) + (a - bb)] -= la * B[(j + bb) * (w + 1) + bb];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) info[s] = bad;
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
  const double* Ls = L + s * M * (w + 1);
  double* rs = r + s * M;
  double* xs = x + s * M;
  for (int64_t i = 0; i < M; ++i) {
    const double* li = Ls + i * (w + 1);
    double acc = 0.0;
    for (int d = 1 + lane; d <= w; d += 32)
      if (i - d >= 0) acc += li[d] * zr[(i - d) & rm];
    acc = warp_sum(acc);
    const double y = (rs[i] - acc) / li[0];
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
      if (i + d < M) acc += Ls[(i + d) * (w + 1) + d] * zr[(i + d) & rm];
    acc = warp_sum(acc);
    const double z = (rs[i] - acc) / Ls[i * (w + 1)];
    __syncwarp();
    if (lane == 0) {
      zr[i & rm] = z;
      xs[i] = mode == 0 ? z : xs[i] + omega * z;
    }
    __syncwarp();
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

int64_t rbws_fn_band_doubles(int count, int c, int planar) {
  const int64_t c1 = c + 1;
  const int64_t nsys = planar ? count * c1 : count;
  const int64_t M = planar ? c1 * c1 : c1 * c1 * c1;
  return nsys * M * (band_w(c, planar) + 1);
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
  band_factor_kernel<<<(unsigned)nsys, 256, 0, St(stream)>>>(nsys, M, band_w(c, planar), band, info);
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
  int ring = 32;
  while (ring < w + 1) ring *= 2;
  const int warps = 4;
  const size_t smem = (size_t)warps * ring * sizeof(double);
  if (smem > 48 * 1024) {
    RBWS_CUDA_CHECK(cudaFuncSetAttribute(band_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
  }
  band_solve_kernel<<<(unsigned)((nsys + warps - 1) / warps), warps * 32, smem, St(stream)>>>(
      nsys, M, w, ring, band, r, x, omega, mode);
  FN_LAUNCHED();
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
