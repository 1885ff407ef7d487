// L1ROC reduced-model kernels (see l1roc.cu).
#pragma once

#include "common.cuh"

namespace rbws {

cudaError_t l1roc_project(int n, int Q, const double* face, const double* node, const double* W,
                          int64_t Wstride, int N, const int64_t* rows, int M, double* Bq,
                          cudaStream_t stream);
cudaError_t l1roc_online(int count, int Q, int M, int N, const double* theta, const double* Bq,
                         const double* bs, int64_t bs_stride, const double* T, double* a,
                         double* c, double* ind, int* status, cudaStream_t stream);
cudaError_t expand(int n, int count, const double* W, int64_t Wstride, int N, const double* a,
                   double* x, cudaStream_t stream);
// out[m][a] = W[a] . v[m] (count x N, dev), per-chunk partials in scratch
size_t basis_dot_scratch(int64_t n3, int count, int N);
cudaError_t basis_dot(int64_t n3, int count, const double* W, int64_t Wstride, int N,
                      const double* v, int64_t vstride, double* out, double* scratch,
                      cudaStream_t stream);
size_t deim_scratch_bytes(int n);
cudaError_t deim_step(int n, const double* W, int64_t Wstride, int N, const double* c,
                      const double* v, const uint8_t* excl, double* col, int64_t* out_idx,
                      double* out_vals, void* scratch, cudaStream_t stream, bool ghosts = true);
cudaError_t dense_solve(int m, const double* A, const double* b, double* x, int* status,
                        cudaStream_t stream);

}  // namespace rbws
