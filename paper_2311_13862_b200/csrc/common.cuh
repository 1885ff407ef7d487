// Shared definitions for the RBWS B200 kernels.
//
// Vector layout ("padded batch layout"): a level with n cells
// per axis stores each parameter instance as an n^3 block of doubles indexed
// i + n*(j + n*k), i,j,k in [0,n).  Interior (free) nodes are i,j,k in
// [1,n-1]; every entry with a zero coordinate is a Dirichlet ghost that stays
// 0.0.  Neighbour addresses of interior nodes that step onto the far
// boundary (coordinate n) wrap onto the next row/plane/instance's ghost
// entries, so stencils need no bounds checks.  A batch of B instances is
// B*n^3 + 2n^2 doubles (a trailing ghost region of two planes, enough for
// the diagonal 27-point / trilinear reads of the last instance's top corner).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define RBWS_HD __host__ __device__ __forceinline__

namespace rbws {

constexpr int kMaxTerms = 8;

// process-wide count of kernel launches issued by this library
void count_launch();
void count_launches(int64_t k);
int64_t launch_count();
// raise fn's dynamic shared-memory limit to `bytes` on the current device (cached per
// kernel and device, thread-safe; no-op at or below the 48 KB default)
cudaError_t smem_attr(const void* fn, size_t bytes);

RBWS_HD int64_t vec_doubles(int n, int batch) {
  return (int64_t)batch * n * n * n + 2 * (int64_t)n * n;
}

// Separable 7-point operator of the finest level.
// face[(q*3+d)*n + i]            : factor of the d-face between nodes i, i+1 along d
// node[((q*3+d)*3+a)*(n+1) + j]  : factor along axis a != d at node j
// theta[mu*Q + q]                : affine weight of term q for instance mu
struct Sep7 {
  int n;
  int Q;
  const double* face;
  const double* node;
  const double* theta;
  int zchg = -1;             // planes where the diagonal changes along z (-1: unknown)
  const int* fz = nullptr;   // [n+1] plane k's diagonal equals plane k-1's (device, host-built)
  const double* wface = nullptr;  // stored +x/+y/+z face weights (3 vectors), or null
  int64_t wstride = 0;
};

// Deterministic reduction of one double per thread over a (possibly 2D)
// block.  Result valid in thread 0.  smem must hold >= 32 doubles.
__device__ __forceinline__ double block_reduce_sum(double v, double* smem) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
  for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
  const int lane = tid & 31, wid = tid >> 5;
  const int nwarps = (nthreads + 31) >> 5;
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (tid == 0) {
    for (int w = 0; w < nwarps; ++w) r += smem[w];
  }
  return r;
}

}  // namespace rbws

#define RBWS_CUDA_CHECK(expr)                                              \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) return rbws_set_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

int rbws_set_error(const char* msg, const char* file, int line);
