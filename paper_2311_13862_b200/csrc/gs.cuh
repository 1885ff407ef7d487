// Batched lexicographic Gauss-Seidel sweeps (the reference's smoother="gs").
#pragma once

#include "stencil.cuh"

namespace rbws {

// One forward (lexicographic) or backward Gauss-Seidel sweep, in place on x, for every
// active instance.  Finest level: the 7-point operator from stored face weights (wface: three
// padded batch vectors at stride wstride); coarse levels: stored 27-point coefficients
// [batch][14][n^3].  b, x: padded batch vectors.
cudaError_t gs7_sweep(int n, int batch, const double* wface, int64_t wstride, const double* b,
                      double* x, bool forward, const LaunchCtx& lc);
cudaError_t gs27_sweep(int n, int batch, const double* coef, const double* b, double* x,
                       bool forward, const LaunchCtx& lc);

}  // namespace rbws
