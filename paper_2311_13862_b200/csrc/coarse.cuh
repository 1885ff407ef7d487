// Matrix-free coarse-level kernels (see coarse.cu).
#pragma once

#include "stencil.cuh"

namespace rbws {

struct CoarseGeom {
  int ty, threads, ytiles, zc, kz;
};
CoarseGeom coarse_geom(int n, int batch, int nz = 0);

// One coarse level's matrix-free operator description.
//   fac:   the level's Kronecker factors [Q*3][3][2][n+1]
//   zsame: [n+1] per-plane flag "z factors equal the previous plane's" (host built)
//   grp:   [3Q] z-group of every term (terms with bitwise identical z factors), G groups
struct CoarseOp {
  int n = 0, Q = 0, G = 0;
  const double* fac = nullptr;
  const int* zsame = nullptr;
  const int* grp = nullptr;
  // per-instance stored 27-point coefficients [batch][14][n^3] (diagonal, 13 forward
  // offsets; symmetric), or null: matrix-free from the factors
  const double* coef = nullptr;
  bool coef_shared = false;  // coef is one coefficient set applied to every instance
  // stored-coefficient hierarchy without per-instance coefficients on this level: the
  // per-term coefficients [Q][14][n^3], combined with theta on the fly (shared by the batch)
  const double* tcoef = nullptr;
  // 1/diag of this level per instance (padded batch), or null (then diag is combined on the fly)
  const double* dinv = nullptr;
};

// mode: 0 apply y=Ax | 1 resid y=b-Ax | 2 jacobi y=x+w(b-Ax)/diag | 4 dinv y=1/diag
cudaError_t coarse_launch(int mode, const CoarseOp& op, const double* theta, int batch,
                          const double* x, const double* b, double* y, double omega,
                          const LaunchCtx& lc);
// stored coefficients of a coarse level (and 1/diag) from its Kronecker factors, for levels
// whose terms fall into more z-groups than the grouped kernel takes
cudaError_t coarse_build_coef(const CoarseOp& op, const double* theta, int batch, double* coef,
                              double* dinv, cudaStream_t stream);
// per-instance coefficients coef[mu] = sum_q theta_q tcoef[q] (and 1/diag) of a stored-coefficient
// level; tcoef = [Q][14][n^3]
// coef may be null: 1/diag only
cudaError_t stored_combine(int n, int Q, const double* tcoef, const double* theta, int batch,
                           double* coef, double* dinv, cudaStream_t stream);
// coarsest level of a stored-coefficient hierarchy: dense operator + Cholesky per instance
cudaError_t coarse_factor_stored(int n0, int Q, const double* tcoef, const double* theta,
                                 int batch, double* L, int* status, cudaStream_t stream);
// finest level of a stored-coefficient hierarchy with batch-shared per-term coefficients:
// z-marching kernel with TMA-staged planes (stored.cu); ok for n in {16,32,64,128}, Q <= 4,
// whole instances (no slab z-ranges)
bool stored_zm_ok(int n, int Q, const LaunchCtx& lc);
cudaError_t stored_zm_launch(int mode, int n, int Q, const double* tcoef, const double* theta,
                             const double* dinv, int batch, const double* x, const double* b, double* y,
                             double omega, const LaunchCtx& lc);
constexpr int kCoarseMaxGroups = 4;  // coarse_kron_kernel<G> instantiations
// coarsest level: dense Galerkin operator from the factors + Cholesky per instance
cudaError_t coarse_factor_kf(int n0, int Q, const double* fac, const double* theta, int batch,
                             double* L, int* status, cudaStream_t stream);

}  // namespace rbws
