// Stencil, transfer and vector kernels of the batched V-cycle / PCG path.
#pragma once

#include "common.cuh"

namespace rbws {

enum StencilMode : int {
  MODE_APPLY = 0,   // y = A x
  MODE_RESID = 1,   // y = b - A x
  MODE_JACOBI = 2,  // y = x + omega (b - A x) / d
  MODE_PRE = 3,     // y = b - A (omega dinv b)     (nu=1 pre-smooth from zero + residual)
  MODE_DINV = 4,    // y = 1 / d
};

enum DotMode : int { DOT_NONE = 0, DOT_XAX = 1, DOT_BY = 2, DOT_YY = 3 };

struct LaunchCtx {
  cudaStream_t stream;
  const int* active;  // per-instance flag (nullptr = all active)
  // z-range of output planes [zlo, zhi) of every instance (0, 0 = the whole grid).  The slab
  // path (slab.cu) passes its owned planes with "virtual" base pointers: a pointer v such
  // that v + k*n^2 is global plane k, valid for the planes a kernel touches (zlo-1 .. zhi).
  int zlo = 0, zhi = 0;
};

// ---- finest level (separable 7-point) -----------------------------------
struct Sep7Geom {
  int tx, ty, zc;     // block dims and z-chunks
  int tiles;          // partial-sum slots per instance
};
Sep7Geom sep7_geom(int n, int batch);

// generic mode kernel; partial (if dot != DOT_NONE) gets tiles doubles per instance
cudaError_t sep7_launch(const Sep7& op, int batch, int mode, int dot, const double* x,
                        const double* b, const double* dinv, double* y, double* partial,
                        double omega, const LaunchCtx& lc);

// ---- transfers -----------------------------------------------------------
// bc = P^T r  (coarse n_c = n_f/2); with dinv_c/uc also uc = omega dinv_c bc
cudaError_t restrict_launch(int nf, int batch, const double* rf, double* bc, const LaunchCtx& lc,
                            const double* dinv_c = nullptr, double* uc = nullptr,
                            double omega = 0.0);
// y pass of a restriction whose x / z passes ran in fine_pre_xz (t: n/2 x n x n/2 per instance)
cudaError_t restrict_y_launch(int nf, int batch, const double* t, double* bc, const LaunchCtx& lc,
                              const double* dinv_c = nullptr, double* uc = nullptr,
                              double omega = 0.0);
// mode 0: u += P e ;  mode 1: u = omega dinv b + P e ;  mode 2: u = b + P e
cudaError_t prolong_launch(int nf, int batch, int mode, const double* ec, double* u,
                           const double* b, const double* dinv, double omega, const LaunchCtx& lc);

// ---- coarsest dense solve ------------------------------------------------
cudaError_t coarse_solve(int n0, int batch, const double* L, const double* b, double* x,
                         const LaunchCtx& lc);

// ---- vector ops ----------------------------------------------------------
// partial[mu*tiles + t] = sum x*y over instance mu (tiles from vec_tiles)
int vec_tiles(int n);
// u = omega dinv b (elementwise, padded batch vectors)
cudaError_t vec_scale_dinv(int n, int batch, double omega, const double* dinv, const double* b,
                           double* u, cudaStream_t stream);
cudaError_t vec_dot(int n, int batch, const double* x, int64_t x_stride, const double* y,
                    int64_t y_stride, double* partial, const LaunchCtx& lc);
// partial[t] = sum x*y over `count` contiguous doubles, (count + 2047)/2048 tiles
cudaError_t vec_dot_range(int64_t count, const double* x, const double* y, double* partial,
                          cudaStream_t stream);

}  // namespace rbws
