// Native runtime of the batched MGCG path: the multigrid hierarchy of a
// separable affine problem (mu-independent), the per-batch context
// (mu-dependent coarse operators, Cholesky factors, work vectors), the
// batched V-cycle and the batched PCG driver.
#pragma once

#include <array>
#include <vector>

#include "coarse.cuh"
#include "stencil.cuh"
#include "tail.cuh"

namespace rbws {

// device -> host copy of control data through mapped pinned memory (no copy engine);
// synchronises the stream
cudaError_t fetch_to_host(void* dst, const void* src, size_t bytes, cudaStream_t stream);

struct Hierarchy {
  int n = 0, m0 = 0, levels = 0, Q = 0;
  std::vector<int> cells;           // coarse (0) .. fine (levels-1)
  double* d_face = nullptr;         // fine separable tables
  double* d_node = nullptr;
  std::vector<double*> d_fac;       // per level 1D Kronecker factors [Q*3][3][2][n+1]
  std::vector<int*> d_zsame;        // per level [n+1]: z factors of plane k == plane k-1
  int* d_fzsame = nullptr;          // finest level [n+1]: same flags for the separable tables
  int fine_zchg = -1;               // finest planes whose diagonal differs from the previous
  std::vector<int*> d_grp;          // per level [3Q]: z-group of every term
  std::vector<int> G;               // per level: number of z-groups
  std::vector<std::vector<double>> h_fac;
  // stored-coefficient hierarchy (assembled FEM problems, rbws_hierarchy_create_stored): every
  // level's operator is sum_q theta_q C_q with per-term symmetric 27-point coefficients
  // d_tcoef[l] = [Q][14][n_l^3] (padded layout, zero on ghosts); no Kronecker factors
  bool stored = false;
  std::vector<double*> d_tcoef;

  ~Hierarchy();
  // the finest level runs the separable 7-point kernels (fine.cu)
  bool sep_fine(int l) const { return !stored && l == levels - 1; }
  CoarseOp coarse_op(int l) const {
    CoarseOp o;
    o.n = cells[l]; o.Q = Q; o.G = G[l];
    o.fac = d_fac[l]; o.zsame = d_zsame[l]; o.grp = d_grp[l];
    if (stored) o.tcoef = d_tcoef[l];
    return o;
  }
};

int kron_factors(int n, int m0, int Q, const double* face, const double* node,
                 std::vector<int>& cells, std::vector<std::vector<double>>& fac);
int hierarchy_create(Hierarchy** out, int n, int m0, int Q, const double* face,
                     const double* node);
// coef: host, levels 0..L-1 concatenated, level l = [Q][14][n_l^3] (n_l = m0 2^l)
int hierarchy_create_stored(Hierarchy** out, int n, int m0, int Q, const double* coef);

struct LevelBuf {
  int n = 0;
  double* b = nullptr;     // level rhs (coarse levels)
  double* e = nullptr;     // level correction (coarse levels)
  double* t1 = nullptr;    // scratch
  double* t2 = nullptr;    // scratch (nu != 1)
  double* t3 = nullptr;    // scratch (nu != 1)
  double* zero = nullptr;  // zeros (nu != 1)
  double* dinv = nullptr;  // 1/diag per instance
  double* coef = nullptr;  // stored 27-point coefficients [cap][14][n^3] (many z-groups)
  double* u = nullptr;     // pre-scaled rhs w D^-1 b (coarse levels 1..L-2, nu=1)
};

// kernel classes timed by the optional event profiler (bench.py roofline)
enum ProfClass : int {
  PROF_FINE_APPLY_DOT = 0,  // p . A p                     (reads p)
  PROF_FINE_CG_UPDATE = 1,  // x += a p, r -= a A p, |r|^2 (reads p x r, writes x r)
  PROF_FINE_PRE = 2,        // r1 = b - A(w D^-1 b)        (reads b dinv, writes r1)
  PROF_FINE_RESTRICT = 3,   // bc = P^T r1
  PROF_FINE_PROLONG = 4,    // u0 = w D^-1 b + P e
  PROF_FINE_POST = 5,       // s = u0 + w (b - A u0)/d, r.s
  PROF_FINE_XPBY = 6,       // p = s + beta p
  PROF_COARSE = 7,          // all coarse levels of one V-cycle
  PROF_SCALARS = 8,         // per-instance scalar kernels
  PROF_NCLASS = 9
};

struct Batch {
  Hierarchy* h = nullptr;
  int cap = 0, count = 0, nu = 1;
  int maxl = 0;                     // levels with buffers (< levels: coarse-only, slab path)
  int smoother = 0;                 // 0 damped Jacobi (isotropic default), 1 Gauss-Seidel ("gs")
  bool fuse_restrict = true;        // finest pre-smoothing + x/z restriction in one kernel
  bool fused_used = false;          // the last V-cycle took the fused path
  bool sw_used = false;             // ... with the scaled-weights pre-smoothing kernels
  bool cgp_used = false;            // the last solve ran the fused CG update (cgp.cu)
  bool pre_done = false;            // the finest pre-smoothing residual + x/z restriction of the
                                    // next V-cycle already ran inside the CG update (cgp.cu)
  double omega = 0.7;
  double* theta = nullptr;          // [cap][Q]
  double* wface = nullptr;          // stored fine face weights [3][cap n^3 + 2n^2] (SCW kernels)
  int64_t wstride = 0;
  std::vector<LevelBuf> lv;
  double* L0 = nullptr;             // coarsest Cholesky factors [cap][m][m]
  int* d_status = nullptr;          // coarse factor status per instance
  // PCG state (fine level)
  double *r = nullptr, *p = nullptr, *p2 = nullptr, *s = nullptr, *t_res = nullptr;
  double* r2 = nullptr;             // second residual buffer (fused CG update, allocated on use)
  double* rcur = nullptr;           // the current residual of the running solve (r or r2)
  double *rs = nullptr, *alpha = nullptr, *beta = nullptr, *scale = nullptr;
  int *active = nullptr, *iters = nullptr, *pstatus = nullptr, *nactive = nullptr;
  int* h_nactive = nullptr;         // pinned
  std::vector<int> h_active, h_sent;  // streaming download bookkeeping (host)
  std::vector<cudaEvent_t> dl_ev;     // compute-stream points the downloads wait for
  std::vector<int> dl_pending;        // marked download calls whose copies are not enqueued yet
  // device-side PCG loop (iterations 1..) as a conditional CUDA graph, cached per solve shape
  bool use_graph = true;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double* gkey_x = nullptr;
  const int* gkey_active = nullptr;
  int gkey_count = 0, gkey_lmax = 0, gkey_hl = 0, gkey_smoother = -1, gkey_fused = -1,
      gkey_variant = -2;
  const double* gkey_wface = nullptr;
  const double* gkey_rcur = nullptr;
  double gkey_delta = 0.0;
  void drop_graph();                // invalidate the cached executable (smoother/graph changes)
  int64_t gbody_launches = 0;
  cudaStream_t gstream = nullptr;     // capture/launch stream when the caller's is the legacy one
  cudaEvent_t gev[2] = {nullptr, nullptr};
  double* partial = nullptr;        // [cap][max tiles]
  double* partial2 = nullptr;
  double* hist = nullptr;           // [cap][hist_len]
  int hist_len = 0;
  int64_t partial_cap = 0;

  bool prof_on = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  std::vector<std::array<int, 4>> recs;
  double prof_ms[PROF_NCLASS] = {0};
  int64_t prof_calls[PROF_NCLASS] = {0};
  int64_t prof_units[PROF_NCLASS] = {0};  // instance-launches (active instances summed)
  int cur_active = 0;                     // host-known active instances
  int prof_begin(cudaStream_t s);
  void prof_end(int cls, int start, cudaStream_t s);
  void prof_flush();

  ~Batch();
  Sep7 fine_op() const;
  CoarseOp cop(int l) const {  // the level's operator with this batch's stored coefficients
    CoarseOp o = h->coarse_op(l);
    o.coef = lv[l].coef;
    o.dinv = lv[l].dinv;
    return o;
  }
  int vcycle(int lvl, const double* b, double* out, double* dot_partial, const LaunchCtx& lc);
  bool tail_level(int lvl, const LaunchCtx& lc) const;  // fused coarse tail (tail.cu)
};

// maxl: allocate levels 0..maxl-1 only (0 = all; the slab path's replicated coarse levels)
int batch_create(Batch** out, Hierarchy* h, int cap, int nu, double omega, int maxl = 0);
int batch_setup(Batch* b, const double* theta, int count, cudaStream_t stream);
// smoother kind (before batch_setup): 1 = Gauss-Seidel, which needs stored fine face weights
// and stored coarse coefficients (allocated here)
int batch_set_smoother(Batch* b, int kind);

struct PcgOut {
  int* iters;          // host [count]
  double* hist;        // host [count][l_max+1] (NaN padded)
  double* true_res;    // host [count]
  int* status;         // host [count]: 0 ok, 1 breakdown (non-SPD), 2 not converged
  // optional streaming download: instance m's padded solution (n^3 doubles) is copied to
  // x_host + m * host_stride on copy_stream as soon as it stops iterating
  double* x_host = nullptr;
  int64_t host_stride = 0;
  cudaStream_t copy_stream = nullptr;
};

// per-instance PCG scalar kernels (one warp per instance; partials summed in fixed order)
cudaError_t pcg_init(int count, const double* pf, int ftiles, int fshared, const double* prr,
                     int tiles, double delta, int l_max, double* scale, double* hist,
                     int hist_len, int* active, int* iters, int* status, int* nactive,
                     cudaStream_t s);
cudaError_t pcg_rs(int count, const double* prs, int tiles, double* rs, const int* active,
                   cudaStream_t s);
cudaError_t pcg_alpha(int count, const double* ppap, int tiles, const double* rs, double* alpha,
                      int* active, int* status, cudaStream_t s);
cudaError_t pcg_check(int count, const double* prr, int tiles, const double* scale, double delta,
                      int l_max, double* hist, int hist_len, int* active, int* iters,
                      int* nactive, cudaStream_t s);
cudaError_t pcg_beta(int count, const double* prs, int tiles, double* rs, double* beta,
                     const int* active, cudaStream_t s);
cudaError_t pcg_true(int count, const double* prr, int tiles, const double* scale, double* out,
                     cudaStream_t s);

int solver_set_tail(int v);  // fused coarse tail: 0 off, else on (process-wide, tests / A-B)
int pcg_solve(Batch* b, const double* f, int64_t f_stride, double* x, double delta, int l_max,
              const PcgOut& out, cudaStream_t stream);
// PCG with the iteration-indexed multispace reduced-basis preconditioner (msrb.cu): basis
// min(k, nbases-1) serves iteration k; W[k]: N[k] padded vectors at stride Wstride[k],
// chol[k]: [count][N[k]][N[k]] lower Cholesky factors of W_k^T A(mu) W_k (all device)
int msrbcg_solve(Batch* b, const double* f, int64_t f_stride, double* x, double delta, int l_max,
                 int nbases, const double* const* W, const int64_t* Wstride, const int* N,
                 const double* const* chol, const PcgOut& out, cudaStream_t stream);

}  // namespace rbws
