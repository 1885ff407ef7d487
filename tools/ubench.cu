// Microbenchmark of z-marching stencil pipelines on padded batch vectors
// (development tool; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2311_13862_b200/csrc/tma.cuh"

using namespace rbws;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// V0: thread per column, global loads, register z-march, 7-pt constant stencil
__global__ void v0(const double* __restrict__ x, double* __restrict__ y, int n, int ty) {
  const int mu = blockIdx.z, j = blockIdx.y * ty + threadIdx.y, i = threadIdx.x;
  const long n2 = (long)n * n, base = (long)mu * n2 * n;
  const long col = base + i + (long)n * j;
  double um = x[col], uc = x[col + n2];
  for (int k = 1; k < n; ++k) {
    const long idx = col + (long)k * n2;
    const double up = __ldg(x + idx + n2);
    const double s = __ldg(x + idx + 1) + __ldg(x + idx - 1) + __ldg(x + idx + n) + __ldg(x + idx - n);
    if (i && j) y[idx] = 6.0 * uc - s - up - um;
    um = uc; uc = up;
  }
}

// V1: TMA ring (S slots, one array, ty+2 rows), constant 7-pt stencil, NPT rows per thread
template <int S, int NPT, int MODE>
__global__ void __launch_bounds__(256) v1(const double* __restrict__ x, double* __restrict__ y, int n, int ty) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = (uint64_t*)smem;
  double* ring = (double*)(smem + 128);
  const int mu = blockIdx.z, j0 = blockIdx.y * ty, tid = threadIdx.x;
  const long n2 = (long)n * n, base = (long)mu * n2 * n;
  const int hsz = (ty + 2) * n;
  if (tid == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); mbar_fence_init(); }
  __syncthreads();
  const int skip = j0 == 0;
  auto issue = [&](int p) {
    const int st = p & (S - 1);
    const uint32_t bytes = (ty + 2 - skip) * n * 8;
    mbar_arrive_expect_tx(&bar[st], bytes);
    bulk_g2s(ring + st * hsz + skip * n, x + base + (long)p * n2 + (long)(j0 - 1 + skip) * n, bytes, &bar[st]);
  };
  if (tid == 0) for (int p = 0; p < S && p <= n; ++p) issue(p);
  const int i = tid % n, rl0 = tid / n, rpp = blockDim.x / n;
  mbar_wait(&bar[0], 0); mbar_wait(&bar[1], 0);
  for (int k = 1; k < n; ++k) {
    mbar_wait(&bar[(k + 1) & (S - 1)], ((k + 1) / S) & 1);
    if (MODE == 1) __syncthreads();
    if (MODE == 1 && tid == 0 && k - 2 >= 0 && k - 2 + S <= n) issue(k - 2 + S);
    const double* X0 = ring + (k & (S - 1)) * hsz;
    const double* XM = ring + ((k - 1) & (S - 1)) * hsz;
    const double* XP = ring + ((k + 1) & (S - 1)) * hsz;
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      const int jl = rl0 + r * rpp, j = j0 + jl, hi = (jl + 1) * n + i;
      const double v = 6.0 * X0[hi] - X0[hi + 1] - X0[hi - 1] - X0[hi + n] - X0[hi - n] - XP[hi] - XM[hi];
      if (i && j) y[base + (long)k * n2 + (long)j * n + i] = v;
    }
    if (MODE == 0) {
      __syncthreads();
      if (tid == 0 && k - 1 + S <= n) issue(k - 1 + S);
    }
  }
}


// V2: TMA ring + separable weights.  WM=1: column constants in registers (5Q), z factors from smem,
// thread per column (NPT=1).  WM=2: per-plane H tables in smem (5Q per row), NPT rows per thread.
template <int S, int NPT, int Q, int WM>
__global__ void __launch_bounds__(256) v2(const double* __restrict__ x, double* __restrict__ y, int n, int ty,
                                          const double* __restrict__ tab) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = (uint64_t*)smem;
  double* zf = (double*)(smem + 128);                 // [n+1][3][Q]
  double* H = zf + (n + 1) * 3 * Q;                   // [2][ty][5Q]
  double* ring = H + 2 * ty * 5 * Q;
  const int mu = blockIdx.z, j0 = blockIdx.y * ty, tid = threadIdx.x;
  const long n2 = (long)n * n, base = (long)mu * n2 * n;
  const int hsz = (ty + 2) * n;
  for (int t = tid; t < (n + 1) * 3 * Q; t += blockDim.x) zf[t] = tab[t % 64] + 0.001 * (t & 7);
  if (tid == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); mbar_fence_init(); }
  __syncthreads();
  const int skip = j0 == 0;
  auto issue = [&](int p) {
    const int st = p & (S - 1);
    const uint32_t bytes = (ty + 2 - skip) * n * 8;
    mbar_arrive_expect_tx(&bar[st], bytes);
    bulk_g2s(ring + st * hsz + skip * n, x + base + (long)p * n2 + (long)(j0 - 1 + skip) * n, bytes, &bar[st]);
  };
  if (tid == 0) for (int p = 0; p < S && p <= n; ++p) issue(p);
  const int i = tid % n, rl0 = tid / n, rpp = blockDim.x / n;
  double c[5][Q];
#pragma unroll
  for (int a = 0; a < 5; ++a)
#pragma unroll
    for (int q = 0; q < Q; ++q) c[a][q] = tab[(a * Q + q + i) & 63] * (1.0 + 0.01 * rl0);
  mbar_wait(&bar[0], 0); mbar_wait(&bar[1], 0);
  double wzm = 1.0;
  for (int k = 1; k < n; ++k) {
    mbar_wait(&bar[(k + 1) & (S - 1)], ((k + 1) / S) & 1);
    if (WM == 2) {
      double* Hk = H + (k & 1) * ty * 5 * Q;
      for (int t = tid; t < ty * 5 * Q; t += blockDim.x) Hk[t] = zf[k * 3 * Q + (t % (3 * Q))] * tab[t & 63];
    }
    __syncthreads();
    if (tid == 0 && k - 2 >= 0 && k - 2 + S <= n) issue(k - 2 + S);
    const double* X0 = ring + (k & (S - 1)) * hsz;
    const double* XM = ring + ((k - 1) & (S - 1)) * hsz;
    const double* XP = ring + ((k + 1) & (S - 1)) * hsz;
    const double* zk = zf + k * 3 * Q;
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      const int jl = rl0 + r * rpp, j = j0 + jl, hi = (jl + 1) * n + i;
      double wxp = 0, wxm = 0, wyp = 0, wym = 0, wzp = 0;
      if (WM == 1) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double zx = zk[q], zy = zk[Q + q], fz = zk[2 * Q + q];
          wxp = fma(c[0][q], zx, wxp); wxm = fma(c[1][q], zx, wxm);
          wyp = fma(c[2][q], zy, wyp); wym = fma(c[3][q], zy, wym); wzp = fma(c[4][q], fz, wzp);
        }
      } else {
        const double* h = H + (k & 1) * ty * 5 * Q + jl * 5 * Q;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          wxp = fma(c[0][q], h[q], wxp); wxm = fma(c[1][q], h[q], wxm);
          wyp = fma(c[2][q], h[Q + q], wyp); wym = fma(c[2][q], h[2 * Q + q], wym);
          wzp = fma(c[4][q], h[3 * Q + q], wzp); wzm = fma(c[4][q], h[4 * Q + q], wzm);
        }
      }
      const double d = wxp + wxm + wyp + wym + wzp + wzm;
      double off = wxp * X0[hi + 1];
      off = fma(wxm, X0[hi - 1], off); off = fma(wyp, X0[hi + n], off); off = fma(wym, X0[hi - n], off);
      off = fma(wzp, XP[hi], off); off = fma(wzm, XM[hi], off);
      if (i && j) y[base + (long)k * n2 + (long)j * n + i] = fma(d, X0[hi], -off);
      if (WM == 1) wzm = wzp;
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64, B = argc > 2 ? atoi(argv[2]) : 1024;
  const long L = (long)B * n * n * n + 2L * n * n;
  double *x, *y;
  CK(cudaMalloc(&x, L * 8)); CK(cudaMalloc(&y, L * 8));
  CK(cudaMemset(x, 0, L * 8)); CK(cudaMemset(y, 0, L * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 16.0 * B * (double)(n - 1) * (n - 1) * (n - 1);
  auto run = [&](const char* name, auto launch) {
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-40s %8.3f ms %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  for (int ty : {4, 8}) {
    char nm[64]; snprintf(nm, 64, "v0 global z-march ty=%d", ty);
    run(nm, [&] { v0<<<dim3(1, n / ty, B), dim3(n, ty)>>>(x, y, n, ty); });
  }
  auto tv1 = [&](auto kern, int S, int npt, const char* tag) {
    const int rpp = 256 / n, ty = rpp * npt;
    const size_t smem = 128 + (size_t)S * (ty + 2) * n * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char nm[80]; snprintf(nm, 80, "v1 tma S=%d npt=%d ty=%d %s smem=%zuK", S, npt, ty, tag, smem / 1024);
    run(nm, [&] { kern<<<dim3(1, n / ty, B), rpp * n, smem>>>(x, y, n, ty); });
  };
  tv1(v1<4, 1, 0>, 4, 1, "late"); tv1(v1<4, 2, 0>, 4, 2, "late"); tv1(v1<4, 4, 0>, 4, 4, "late");
  tv1(v1<8, 1, 0>, 8, 1, "late"); tv1(v1<8, 2, 0>, 8, 2, "late"); tv1(v1<8, 4, 0>, 8, 4, "late");
  tv1(v1<8, 1, 1>, 8, 1, "early"); tv1(v1<8, 2, 1>, 8, 2, "early"); tv1(v1<8, 4, 1>, 8, 4, "early");
  tv1(v1<16, 1, 1>, 16, 1, "early"); tv1(v1<16, 2, 1>, 16, 2, "early");
  double* tab; CK(cudaMalloc(&tab, 64 * 8)); CK(cudaMemset(tab, 0, 64 * 8));
  auto tv2 = [&](auto kern, int S, int npt, int Q, const char* tag) {
    const int rpp = 256 / n, ty = rpp * npt;
    const size_t smem = 128 + (size_t)((n + 1) * 3 * Q + 2 * ty * 5 * Q) * 8 + (size_t)S * (ty + 2) * n * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char nm[80]; snprintf(nm, 80, "v2 %s S=%d npt=%d Q=%d smem=%zuK", tag, S, npt, Q, smem / 1024);
    run(nm, [&] { kern<<<dim3(1, n / ty, B), rpp * n, smem>>>(x, y, n, ty, tab); });
  };
  tv2(v2<8, 1, 4, 1>, 8, 1, 4, "colconst"); tv2(v2<8, 1, 8, 1>, 8, 1, 8, "colconst");
  tv2(v2<16, 1, 4, 1>, 16, 1, 4, "colconst");
  tv2(v2<8, 1, 4, 2>, 8, 1, 4, "Htable"); tv2(v2<8, 2, 4, 2>, 8, 2, 4, "Htable");
  tv2(v2<8, 2, 8, 2>, 8, 2, 8, "Htable");
  run("cudaMemcpy d2d", [&] { cudaMemcpyAsync(y, x, (long)B * n * n * n * 8, cudaMemcpyDeviceToDevice); });
  return 0;
}
