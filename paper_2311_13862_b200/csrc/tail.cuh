// Fused coarse tail of the V-cycle (see tail.cu).
#pragma once

#include "coarse.cuh"

namespace rbws {

constexpr int kTailMaxLevels = 4;  // smoothed levels 1 .. LT fused with the coarsest solve

struct TailArgs {
  int LT = 0;                               // top fused level (>= 1)
  int Q = 0;
  int n[kTailMaxLevels + 1] = {};           // cells per axis of levels 0 .. LT
  const double* fac[kTailMaxLevels + 1] = {};  // Kronecker factors per level [Q*3][3][2][n+1]
  const int* grp[kTailMaxLevels + 1] = {};     // z-group of every term per level [3Q]
  const double* theta = nullptr;            // [batch][Q]
  const double* b = nullptr;                // level-LT rhs (padded batch)
  const double* u = nullptr;                // level-LT pre-scaled rhs w D^-1 b
  double* e = nullptr;                      // level-LT correction (out)
  const double* L0 = nullptr;               // coarsest Cholesky factors [batch][m][m]
  const int* active = nullptr;
  double omega = 0.0;
};

// levels 1 .. LT have at most 16 cells per axis, G z-groups each, and fit shared memory
bool coarse_tail_fits(const TailArgs& a, int G);
// one V-cycle from zero on level LT for every active instance: e = V(b) (nu = 1, damped Jacobi)
cudaError_t coarse_tail_launch(const TailArgs& a, int G, int batch, cudaStream_t stream);

}  // namespace rbws
