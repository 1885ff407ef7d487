// Batched PCG with the iteration-indexed multispace reduced-basis preconditioner
// (reference msrbcg_solve, msrb.py:152-170; MsrbPreconditioner.__call__, msrb.py:77-85; the
// PCG recurrence of krylov.py:42-109).  One native loop for the whole batch: per-instance
// scalars and the active set stay on the device (one readback of the active count per
// iteration), every vector operation is a kernel of this library:
//   s = P_k(r):  u = one symmetric Gauss-Seidel sweep from zero on r   (gs7_sweep / gs27_sweep)
//                res = r - A u                                          (fine_resid / coarse_launch)
//                t = W_k^T res                                          (basis_dot)
//                t = (W_k^T A W_k)^{-1} t from the per-instance Cholesky factor (chol_solve)
//                s = u + W_k t                                          (expand + add)
// The bases W_k and the factors of the reduced operators are set up by the caller
// (msrb.py: POD + W^T A_q W projections, theta-combined and factored per instance).
#include <algorithm>
#include <cstring>
#include <vector>

#include "coarse.cuh"
#include "fine.cuh"
#include "gs.cuh"
#include "l1roc.cuh"
#include "solver.cuh"

int rbws_set_error(const char* msg, const char* file, int line);
#define RBWS_FAIL(msg) return rbws_set_error(msg, __FILE__, __LINE__)

namespace rbws {

// one warp per instance: t <- (L L^T)^{-1} t, L lower-triangular row-major [N][N] (N <= 64)
__global__ void __launch_bounds__(128) msrb_chol_solve_kernel(int count, int N,
                                                              const double* __restrict__ Lall,
                                                              double* __restrict__ t,
                                                              const int* __restrict__ active) {
  __shared__ double ysh[4][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mu = blockIdx.x * 4 + warp;
  if (mu >= count) return;
  if (active && !active[mu]) return;
  const double* L = Lall + (int64_t)mu * N * N;
  double* y = ysh[warp];
  for (int r = lane; r < N; r += 32) y[r] = t[(int64_t)mu * N + r];
  __syncwarp();
  for (int r = 0; r < N; ++r) {  // L y = t
    double s = 0.0;
    for (int c = lane; c < r; c += 32) s = fma(L[r * N + c], y[c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = (y[r] - s) / L[r * N + r];
    __syncwarp();
  }
  for (int r = N - 1; r >= 0; --r) {  // L^T x = y
    double s = 0.0;
    for (int c = r + 1 + lane; c < N; c += 32) s = fma(L[c * N + r], y[c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = (y[r] - s) / L[r * N + r];
    __syncwarp();
  }
  for (int r = lane; r < N; r += 32) t[(int64_t)mu * N + r] = y[r];
}

// elementwise kernels over the n^3 entries of every active instance
__global__ void __launch_bounds__(256) msrb_add_kernel(int64_t n3, double* __restrict__ s,
                                                       const double* __restrict__ w,
                                                       const int* __restrict__ active) {
  const int mu = blockIdx.y;
  if (active && !active[mu]) return;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const int64_t o = (int64_t)mu * n3 + X;
  s[o] += w[o];
}

__global__ void __launch_bounds__(256) msrb_xpby_kernel(int64_t n3, const double* __restrict__ s,
                                                        const double* __restrict__ beta,
                                                        double* __restrict__ p,
                                                        const int* __restrict__ active) {
  const int mu = blockIdx.y;
  if (!active[mu]) return;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const int64_t o = (int64_t)mu * n3 + X;
  p[o] = beta ? fma(beta[mu], p[o], s[o]) : s[o];
}

__global__ void __launch_bounds__(256) msrb_update_kernel(int64_t n3, const double* __restrict__ p,
                                                          const double* __restrict__ Ap,
                                                          const double* __restrict__ alpha,
                                                          double* __restrict__ x,
                                                          double* __restrict__ r,
                                                          const int* __restrict__ active) {
  const int mu = blockIdx.y;
  if (!active[mu]) return;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const int64_t o = (int64_t)mu * n3 + X;
  const double a = alpha[mu];
  x[o] = fma(a, p[o], x[o]);
  r[o] = fma(-a, Ap[o], r[o]);
}

int msrbcg_solve(Batch* b, const double* f, int64_t f_stride, double* x, double delta, int l_max,
                 int nbases, const double* const* W, const int64_t* Wstride, const int* N,
                 const double* const* chol, const PcgOut& out, cudaStream_t stream) {
  if (!(delta > 0)) RBWS_FAIL("tolerance must be positive");
  if (l_max < 0) RBWS_FAIL("l_max must be non-negative");
  Hierarchy* h = b->h;
  const int count = b->count, n = h->n, L = h->levels;
  if (count < 1) RBWS_FAIL("batch_setup must be called before solving");
  if (b->maxl < L) RBWS_FAIL("msrbcg needs the finest-level buffers");
  const bool fine = h->sep_fine(L - 1);
  if (fine ? !b->wface : !b->lv[L - 1].coef)
    RBWS_FAIL("msrbcg needs a batch with smoother = 1 (Gauss-Seidel sweeps on stored weights)");
  if (nbases < 0) RBWS_FAIL("nbases must be non-negative");
  int nmax = 0;
  for (int k = 0; k < nbases; ++k) {
    if (N[k] < 0 || N[k] > 64) RBWS_FAIL("basis dimension must be in [0, 64]");
    if (N[k] > 0 && (!W[k] || !chol[k])) RBWS_FAIL("null basis / factor");
    nmax = std::max(nmax, N[k]);
  }
  const int64_t n3 = (int64_t)n * n * n;
  if (f_stride != 0 && f_stride != n3) RBWS_FAIL("f_stride must be 0 (shared rhs) or n^3");
  const int hist_len = l_max + 1;
  cudaError_t e = cudaSuccess;
  if (hist_len > b->hist_len || !b->hist) {
    cudaFree(b->hist);
    b->hist = nullptr;
    e = cudaMalloc((void**)&b->hist, sizeof(double) * (size_t)b->cap * hist_len);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    b->hist_len = hist_len;
  }
  const int hl = b->hist_len;
  const int tiles = vec_tiles(n);
  double* tbuf = nullptr;     // [count][nmax] reduced coefficients
  double* scratch = nullptr;  // basis_dot partials
  if (nmax > 0) {
    e = cudaMalloc((void**)&tbuf, sizeof(double) * (size_t)count * nmax);
    if (e == cudaSuccess) e = cudaMalloc((void**)&scratch, basis_dot_scratch(n3, count, nmax));
    if (e != cudaSuccess) { cudaFree(tbuf); RBWS_FAIL(cudaGetErrorString(e)); }
  }
  struct Guard {  // (cudaFree synchronises: the solve's host readbacks are done by then)
    double *a, *b;
    ~Guard() { cudaFree(a); cudaFree(b); }
  } guard{tbuf, scratch};

  LaunchCtx all{stream, nullptr};
  LaunchCtx act{stream, b->active};
  const dim3 vg((unsigned)((n3 + 255) / 256), count);
  const Sep7 fop = fine ? b->fine_op() : Sep7{};
  const CoarseOp cop = fine ? CoarseOp{} : b->cop(L - 1);
  // y = rhs - A v (rhs stride rs) / y = A v, for the whole batch or the active instances
  auto resid = [&](const double* v, const double* rhs, bool shared, double* y,
                   const LaunchCtx& lc) -> cudaError_t {
    if (fine) return fine_resid(fop, count, v, rhs, y, nullptr, lc, shared);
    if (shared) return cudaErrorInvalidValue;
    return coarse_launch(1, cop, b->theta, count, v, rhs, y, 0.0, lc);
  };
  auto apply = [&](const double* v, double* y, const LaunchCtx& lc) -> cudaError_t {
    if (fine) return fine_apply(fop, count, v, y, nullptr, lc);
    return coarse_launch(0, cop, b->theta, count, v, nullptr, y, 0.0, lc);
  };
  const bool fshared = (f_stride == 0);
  if (fshared && !fine) RBWS_FAIL("stored-coefficient problems take one rhs per instance");
  double* u = b->s;                 // the preconditioned residual is built in place
  double* res = b->p2;              // r - A u
  double* wt = b->lv[L - 1].t1;     // W t
  auto precond = [&](int k) -> cudaError_t {  // b->s = P_k(b->r) for the active instances
    cudaError_t ee = cudaMemsetAsync(u, 0, sizeof(double) * count * n3, stream);
    for (int pass = 0; pass < 2 && ee == cudaSuccess; ++pass)
      ee = fine ? gs7_sweep(n, count, b->wface, b->wstride, b->r, u, pass == 0, act)
                : gs27_sweep(n, count, b->lv[L - 1].coef, b->r, u, pass == 0, act);
    if (ee != cudaSuccess || nbases == 0) return ee;
    const int kb = std::min(k, nbases - 1);
    if (N[kb] == 0) return ee;
    ee = resid(u, b->r, false, res, act);
    if (ee == cudaSuccess)
      ee = basis_dot(n3, count, W[kb], Wstride[kb], N[kb], res, n3, tbuf, scratch, stream);
    if (ee != cudaSuccess) return ee;
    count_launch();
    msrb_chol_solve_kernel<<<(count + 3) / 4, 128, 0, stream>>>(count, N[kb], chol[kb], tbuf,
                                                                b->active);
    ee = expand(n, count, W[kb], Wstride[kb], N[kb], tbuf, wt, stream);
    if (ee != cudaSuccess) return ee;
    count_launch();
    msrb_add_kernel<<<vg, 256, 0, stream>>>(n3, u, wt, b->active);
    return cudaGetLastError();
  };

  e = vec_dot(n, fshared ? 1 : count, f, f_stride, f, f_stride, b->partial2, all);
  if (e == cudaSuccess) e = resid(x, f, fshared, b->r, all);
  if (e == cudaSuccess) e = vec_dot(n, count, b->r, n3, b->r, n3, b->partial, all);
  if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
  if (e == cudaSuccess)
    e = pcg_init(count, b->partial2, tiles, fshared ? 1 : 0, b->partial, tiles, delta, l_max,
                 b->scale, b->hist, hl, b->active, b->iters, b->pstatus, b->nactive, stream);
  if (e == cudaSuccess) e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  if (*b->h_nactive > 0) {
    e = precond(0);
    if (e == cudaSuccess) e = vec_dot(n, count, b->r, n3, b->s, n3, b->partial, act);
    if (e == cudaSuccess) e = pcg_rs(count, b->partial, tiles, b->rs, b->active, stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    const double* beta = nullptr;
    for (int k = 0; k < l_max; ++k) {
      count_launch();
      msrb_xpby_kernel<<<vg, 256, 0, stream>>>(n3, b->s, beta, b->p, b->active);
      e = apply(b->p, b->t_res, act);
      if (e == cudaSuccess) e = vec_dot(n, count, b->p, n3, b->t_res, n3, b->partial, act);
      if (e == cudaSuccess)
        e = pcg_alpha(count, b->partial, tiles, b->rs, b->alpha, b->active, b->pstatus, stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      count_launch();
      msrb_update_kernel<<<vg, 256, 0, stream>>>(n3, b->p, b->t_res, b->alpha, x, b->r, b->active);
      e = vec_dot(n, count, b->r, n3, b->r, n3, b->partial, act);
      if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
      if (e == cudaSuccess)
        e = pcg_check(count, b->partial, tiles, b->scale, delta, l_max, b->hist, hl, b->active,
                      b->iters, b->nactive, stream);
      if (e == cudaSuccess) e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      if (*b->h_nactive == 0) break;
      e = precond(k + 1);
      if (e == cudaSuccess) e = vec_dot(n, count, b->r, n3, b->s, n3, b->partial, act);
      if (e == cudaSuccess) e = pcg_beta(count, b->partial, tiles, b->rs, b->beta, b->active, stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      beta = b->beta;
    }
  }
  // true residual of every instance, reports to the host
  e = resid(x, f, fshared, b->t_res, all);
  if (e == cudaSuccess) e = vec_dot(n, count, b->t_res, n3, b->t_res, n3, b->partial, all);
  double* d_true = b->beta;
  if (e == cudaSuccess) e = pcg_true(count, b->partial, tiles, b->scale, d_true, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  std::vector<double> hh((size_t)count * hl);
  e = fetch_to_host(hh.data(), b->hist, sizeof(double) * count * hl, stream);
  if (e == cudaSuccess && out.iters) e = fetch_to_host(out.iters, b->iters, sizeof(int) * count, stream);
  if (e == cudaSuccess && out.true_res)
    e = fetch_to_host(out.true_res, d_true, sizeof(double) * count, stream);
  if (e == cudaSuccess && out.status)
    e = fetch_to_host(out.status, b->pstatus, sizeof(int) * count, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  if (out.hist)
    for (int m = 0; m < count; ++m)
      memcpy(out.hist + (size_t)m * hist_len, hh.data() + (size_t)m * hl, sizeof(double) * hist_len);
  if (out.status && out.true_res)
    for (int m = 0; m < count; ++m)
      if (!(out.status[m] & 1) && !(out.true_res[m] <= delta)) out.status[m] |= 2;
  return 0;
}

}  // namespace rbws
