// extern "C" boundary (include/rbws_b200.h).
#include "../../include/rbws_b200.h"
#include "coarse.cuh"
#include "fine.cuh"
#include "gs.cuh"
#include "l1roc.cuh"
#include "slab.cuh"
#include "solver.cuh"

const char* rbws_get_error();

#define RBWS_FAIL(msg) return rbws_set_error(msg, __FILE__, __LINE__)
#define RBWS_CHECK(expr)                                                          \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) return rbws_set_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

using rbws::Batch;
using rbws::Hierarchy;

static inline Hierarchy* H(rbws_hierarchy* h) { return reinterpret_cast<Hierarchy*>(h); }
static inline const Hierarchy* H(const rbws_hierarchy* h) { return reinterpret_cast<const Hierarchy*>(h); }
static inline Batch* B(rbws_batch* b) { return reinterpret_cast<Batch*>(b); }
static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int rbws_version(void) { return 100; }

const char* rbws_last_error(void) { return rbws_get_error(); }

int64_t rbws_launch_count(void) { return rbws::launch_count(); }

int rbws_fetch(void* dst_host, const void* src_device, int64_t bytes, void* stream) {
  if (bytes < 0) RBWS_FAIL("negative byte count");
  RBWS_CHECK(rbws::fetch_to_host(dst_host, src_device, (size_t)bytes, S(stream)));
  return 0;
}

int rbws_hierarchy_create(rbws_hierarchy** out, int n, int m0, int nterms, const double* face,
                          const double* node) {
  if (!out || !face || !node) RBWS_FAIL("null argument");
  Hierarchy* h = nullptr;
  if (rbws::hierarchy_create(&h, n, m0, nterms, face, node)) return 1;
  *out = reinterpret_cast<rbws_hierarchy*>(h);
  return 0;
}

int rbws_hierarchy_create_stored(rbws_hierarchy** out, int n, int m0, int nterms,
                                 const double* coef) {
  if (!out || !coef) RBWS_FAIL("null argument");
  Hierarchy* h = nullptr;
  if (rbws::hierarchy_create_stored(&h, n, m0, nterms, coef)) return 1;
  *out = reinterpret_cast<rbws_hierarchy*>(h);
  return 0;
}

int rbws_hierarchy_is_stored(const rbws_hierarchy* h) { return H(h)->stored ? 1 : 0; }

int rbws_hierarchy_term_apply(const rbws_hierarchy* h, int level, int term, int count,
                              const double* x, double* y, void* stream) {
  const Hierarchy* hh = H(h);
  if (!hh->stored) RBWS_FAIL("term products need a stored-coefficient hierarchy");
  if (level < 0 || level >= hh->levels) RBWS_FAIL("level outside hierarchy");
  if (term < 0 || term >= hh->Q) RBWS_FAIL("term outside [0, nterms)");
  if (count < 1) RBWS_FAIL("count must be positive");
  rbws::CoarseOp op;
  op.n = hh->cells[level];
  op.Q = hh->Q;
  const int64_t n3 = (int64_t)op.n * op.n * op.n;
  op.coef = hh->d_tcoef[level] + (int64_t)term * 14 * n3;
  op.coef_shared = true;
  rbws::LaunchCtx lc{S(stream), nullptr};
  RBWS_CHECK(rbws::coarse_launch(0, op, nullptr, count, x, nullptr, y, 0.0, lc));
  return 0;
}

int rbws_hierarchy_destroy(rbws_hierarchy* h) {
  delete H(h);
  return 0;
}

int rbws_hierarchy_levels(const rbws_hierarchy* h) { return H(h)->levels; }

int rbws_hierarchy_cells(const rbws_hierarchy* h, int level) {
  if (level < 0 || level >= H(h)->levels) return -1;
  return H(h)->cells[level];
}

int rbws_hierarchy_factors(const rbws_hierarchy* h, int level, double* out, int64_t capacity) {
  const Hierarchy* hh = H(h);
  if (level < 0 || level >= hh->levels) RBWS_FAIL("level outside hierarchy");
  const auto& f = hh->h_fac[level];
  if ((int64_t)f.size() > capacity) RBWS_FAIL("output buffer too small");
  for (size_t i = 0; i < f.size(); ++i) out[i] = f[i];
  return 0;
}

int rbws_kron_factors(int n, int m0, int nterms, const double* face, const double* node,
                      int level, double* out, int64_t capacity) {
  std::vector<int> cells;
  std::vector<std::vector<double>> fac;
  if (rbws::kron_factors(n, m0, nterms, face, node, cells, fac)) return 1;
  if (level < 0 || level >= (int)cells.size()) RBWS_FAIL("level outside hierarchy");
  if ((int64_t)fac[level].size() > capacity) RBWS_FAIL("output buffer too small");
  for (size_t i = 0; i < fac[level].size(); ++i) out[i] = fac[level][i];
  return 0;
}

int rbws_batch_create(rbws_batch** out, rbws_hierarchy* h, int capacity, int nu, double omega) {
  if (!out || !h) RBWS_FAIL("null argument");
  Batch* b = nullptr;
  if (rbws::batch_create(&b, H(h), capacity, nu, omega)) return 1;
  *out = reinterpret_cast<rbws_batch*>(b);
  return 0;
}

int rbws_batch_destroy(rbws_batch* b) {
  delete B(b);
  return 0;
}

int rbws_batch_set_smoother(rbws_batch* b, int kind) {
  if (!b) RBWS_FAIL("null batch");
  return rbws::batch_set_smoother(B(b), kind);
}

int rbws_smooth(rbws_batch* b, int level, int kind, double* x, const double* rhs, void* stream) {
  Batch* bb = B(b);
  Hierarchy* h = bb->h;
  if (level < 1 || level >= h->levels) RBWS_FAIL("level must be in [1, levels)");
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  if (kind != 1 && kind != 2 && kind != 3) RBWS_FAIL("kind: 1 forward, 2 backward, 3 symmetric GS");
  const int n = h->cells[level];
  rbws::LaunchCtx lc{S(stream), nullptr};
  const bool fine = h->sep_fine(level);
  if (fine ? !bb->wface : !bb->lv[level].coef)
    RBWS_FAIL("Gauss-Seidel sweeps need a batch with smoother = 1 (rbws_batch_set_smoother)");
  for (int pass = 0; pass < 2; ++pass) {
    const bool fwd = (pass == 0);
    if ((fwd && kind == 2) || (!fwd && kind == 1)) continue;
    RBWS_CHECK(fine ? rbws::gs7_sweep(n, bb->count, bb->wface, bb->wstride, rhs, x, fwd, lc)
                    : rbws::gs27_sweep(n, bb->count, bb->lv[level].coef, rhs, x, fwd, lc));
  }
  return 0;
}

int rbws_batch_stored_weights(const rbws_batch* b) {
  return reinterpret_cast<const Batch*>(b)->wface ? 1 : 0;
}

int rbws_batch_fused_restrict(const rbws_batch* b) {
  return reinterpret_cast<const Batch*>(b)->fused_used ? 1 : 0;
}

int rbws_batch_pre_scaled(const rbws_batch* b) {
  return reinterpret_cast<const Batch*>(b)->sw_used ? 1 : 0;
}

int rbws_batch_cg_fused(const rbws_batch* b) {
  return reinterpret_cast<const Batch*>(b)->cgp_used ? 1 : 0;
}

int rbws_batch_set_graph(rbws_batch* b, int enable) {
  if (!b) RBWS_FAIL("null batch");
  if (!enable) B(b)->drop_graph();
  B(b)->use_graph = enable != 0;
  return 0;
}

int rbws_set_kernel_variant(int which, int value) {
  if (which == 0) {
    if (rbws::fine_set_dc(value)) RBWS_FAIL("DC variant must be -1 (auto), 0 or 1");
    return 0;
  }
  if (which == 4) {
    if (rbws::fine_set_cgp(value)) RBWS_FAIL("fused CG update variant must be -1 (auto), 0 or 1");
    return 0;
  }
  if (which == 3) {
    if (rbws::fine_set_direct(value)) RBWS_FAIL("direct p-update variant must be -1 (auto), 0 or 1");
    return 0;
  }
  if (which == 2) {
    if (rbws::solver_set_tail(value)) RBWS_FAIL("tail variant must be -1 (auto), 0 or 1");
    return 0;
  }
  if (which == 1) {
    if (rbws::fine_set_sw(value)) RBWS_FAIL("SW variant must be -1 (auto), 0 or 1");
    return 0;
  }
  RBWS_FAIL("unknown kernel variant");
}

int rbws_batch_setup(rbws_batch* b, const double* theta, int count, int* n_bad, void* stream) {
  Batch* bb = B(b);
  if (rbws::batch_setup(bb, theta, count, S(stream))) return 1;
  if (n_bad) {
    std::vector<int> st(count);
    RBWS_CHECK(rbws::fetch_to_host(st.data(), bb->d_status, sizeof(int) * count, S(stream)));
    int bad = 0;
    for (int v : st) bad += v ? 1 : 0;
    *n_bad = bad;
  }
  return 0;
}

int rbws_apply(rbws_batch* b, int level, const double* x, double* y, void* stream) {
  Batch* bb = B(b);
  Hierarchy* h = bb->h;
  if (level < 0 || level >= h->levels) RBWS_FAIL("level outside hierarchy");
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  rbws::LaunchCtx lc{S(stream), nullptr};
  if (h->sep_fine(level)) {
    RBWS_CHECK(rbws::fine_apply(bb->fine_op(), bb->count, x, y, nullptr, lc));
  } else {
    RBWS_CHECK(rbws::coarse_launch(0, bb->cop(level), bb->theta, bb->count, x, nullptr, y, 0.0, lc));
  }
  return 0;
}

int rbws_jacobi_sweep(rbws_batch* b, int level, const double* x, const double* rhs, double* y,
                      void* stream) {
  Batch* bb = B(b);
  Hierarchy* h = bb->h;
  if (level < 1 || level >= h->levels) RBWS_FAIL("smoothing level must be in [1, levels)");
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  rbws::LaunchCtx lc{S(stream), nullptr};
  if (h->sep_fine(level)) {
    RBWS_CHECK(rbws::fine_jacobi(bb->fine_op(), bb->count, x, rhs, y, bb->omega, nullptr, lc));
  } else {
    RBWS_CHECK(rbws::coarse_launch(2, bb->cop(level), bb->theta, bb->count, x, rhs, y, bb->omega, lc));
  }
  return 0;
}

int rbws_restrict(int nf, int count, const double* rf, double* bc, void* stream) {
  if (nf < 4 || (nf & 1)) RBWS_FAIL("fine grid must have an even number of cells >= 4");
  rbws::LaunchCtx lc{S(stream), nullptr};
  RBWS_CHECK(rbws::restrict_launch(nf, count, rf, bc, lc));
  return 0;
}

int rbws_prolong_add(int nf, int count, const double* ec, double* u, void* stream) {
  if (nf < 4 || (nf & 1)) RBWS_FAIL("fine grid must have an even number of cells >= 4");
  rbws::LaunchCtx lc{S(stream), nullptr};
  RBWS_CHECK(rbws::prolong_launch(nf, count, 0, ec, u, nullptr, nullptr, 0.0, lc));
  return 0;
}

int rbws_vcycle(rbws_batch* b, const double* rhs, double* out, void* stream) {
  Batch* bb = B(b);
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  rbws::LaunchCtx lc{S(stream), nullptr};
  return bb->vcycle(bb->h->levels - 1, rhs, out, nullptr, lc);
}

int rbws_mgcg_solve(rbws_batch* b, const double* f, int64_t f_stride, double* x, double delta,
                    int l_max, int* iters, double* hist, double* true_res, int* status,
                    void* stream) {
  rbws::PcgOut o{iters, hist, true_res, status};
  return rbws::pcg_solve(B(b), f, f_stride, x, delta, l_max, o, S(stream));
}

int rbws_msrbcg_solve(rbws_batch* b, const double* f, int64_t f_stride, double* x, double delta,
                      int l_max, int nbases, const double* const* W, const int64_t* Wstride,
                      const int* N, const double* const* chol, int* iters, double* hist,
                      double* true_res, int* status, void* stream) {
  if (!b || !f || !x) RBWS_FAIL("null argument");
  if (nbases > 0 && (!W || !Wstride || !N || !chol)) RBWS_FAIL("null basis arrays");
  rbws::PcgOut o{iters, hist, true_res, status};
  return rbws::msrbcg_solve(B(b), f, f_stride, x, delta, l_max, nbases, W, Wstride, N, chol, o,
                            S(stream));
}

int rbws_mgcg_solve_to_host(rbws_batch* b, const double* f, int64_t f_stride, double* x,
                            double delta, int l_max, int* iters, double* hist, double* true_res,
                            int* status, void* stream, double* x_host, int64_t host_stride,
                            void* copy_stream) {
  if (!x_host) RBWS_FAIL("null host buffer");
  if (host_stride < 0) RBWS_FAIL("negative host stride");
  const int64_t n = B(b)->h->n;
  if (host_stride < n * n * n) RBWS_FAIL("host stride smaller than one padded instance");
  rbws::PcgOut o{iters, hist, true_res, status};
  o.x_host = x_host;
  o.host_stride = host_stride;
  o.copy_stream = S(copy_stream);
  return rbws::pcg_solve(B(b), f, f_stride, x, delta, l_max, o, S(stream));
}

int rbws_level_kernel(rbws_batch* b, int level, int mode, const double* x, const double* rhs,
                      double* y, void* stream) {
  Batch* bb = B(b);
  Hierarchy* h = bb->h;
  if (level < 1 || level >= h->levels) RBWS_FAIL("level must be in [1, levels)");
  if (mode < 0 || mode > 3) RBWS_FAIL("mode must be 0 apply, 1 resid, 2 jacobi, 3 pre");
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  rbws::LaunchCtx lc{S(stream), nullptr};
  const double* dinv = bb->lv[level].dinv;
  if (h->sep_fine(level)) {
    const rbws::Sep7 op = bb->fine_op();
    cudaError_t e;
    if (mode == 0) e = rbws::fine_apply(op, bb->count, x, y, nullptr, lc);
    else if (mode == 1) e = rbws::fine_resid(op, bb->count, x, rhs, y, nullptr, lc);
    else if (mode == 2) e = rbws::fine_jacobi(op, bb->count, x, rhs, y, bb->omega, nullptr, lc);
    else e = rbws::fine_pre(op, bb->count, rhs, dinv, y, bb->omega, lc);
    RBWS_CHECK(e);
  } else if (mode == 3) {  // pre-smoothing residual = residual of u = w D^-1 rhs
    const int n = h->cells[level];
    RBWS_CHECK(rbws::vec_scale_dinv(n, bb->count, bb->omega, dinv, rhs, bb->lv[level].u, S(stream)));
    RBWS_CHECK(rbws::coarse_launch(1, bb->cop(level), bb->theta,
                                   bb->count, bb->lv[level].u, rhs, y, bb->omega, lc));
  } else {
    RBWS_CHECK(rbws::coarse_launch(mode, bb->cop(level), bb->theta, bb->count, x, rhs, y, bb->omega,
                                   lc));
  }
  return 0;
}

int rbws_batch_dinv(rbws_batch* b, int level, double* out, void* stream) {
  Batch* bb = B(b);
  if (level < 1 || level >= bb->h->levels) RBWS_FAIL("level must be in [1, levels)");
  if (bb->count < 1) RBWS_FAIL("batch_setup must be called first");
  const int n = bb->h->cells[level];
  RBWS_CHECK(cudaMemcpyAsync(out, bb->lv[level].dinv,
                             sizeof(double) * rbws::vec_doubles(n, bb->count),
                             cudaMemcpyDeviceToDevice, S(stream)));
  return 0;
}

int rbws_batch_profile(rbws_batch* b, int enable) {
  Batch* bb = B(b);
  bb->prof_on = enable != 0;
  for (int k = 0; k < rbws::PROF_NCLASS; ++k) {
    bb->prof_ms[k] = 0.0;
    bb->prof_calls[k] = 0;
    bb->prof_units[k] = 0;
  }
  return 0;
}

int rbws_batch_profile_read(rbws_batch* b, double* ms, int64_t* calls, int64_t* units,
                            int nclass) {
  Batch* bb = B(b);
  for (int k = 0; k < nclass && k < rbws::PROF_NCLASS; ++k) {
    ms[k] = bb->prof_ms[k];
    calls[k] = bb->prof_calls[k];
    units[k] = bb->prof_units[k];
  }
  return 0;
}

int rbws_l1roc_project(rbws_hierarchy* h, const double* W, int64_t Wstride, int N,
                       const int64_t* rows, int M, double* Bq, void* stream) {
  if (H(h)->stored) RBWS_FAIL("stored-coefficient problems project with rbws_hierarchy_term_apply");
  Hierarchy* hh = H(h);
  RBWS_CHECK(rbws::l1roc_project(hh->n, hh->Q, hh->d_face, hh->d_node, W, Wstride, N, rows, M, Bq,
                                 S(stream)));
  return 0;
}

int rbws_l1roc_online(int count, int Q, int M, int N, const double* theta, const double* Bq,
                      const double* bs, int64_t bs_stride, const double* T, double* a, double* c,
                      double* ind, int* status, void* stream) {
  if (count < 1 || N < 1 || M < N) RBWS_FAIL("need count >= 1 and M >= N >= 1");
  RBWS_CHECK(rbws::l1roc_online(count, Q, M, N, theta, Bq, bs, bs_stride, T, a, c, ind, status,
                                S(stream)));
  return 0;
}

int rbws_basis_dot(int64_t n3, int count, const double* W, int64_t Wstride, int N,
                   const double* v, int64_t vstride, double* out, void* stream) {
  if (N < 1 || count < 1 || n3 < 1) RBWS_FAIL("empty projection");
  void* scratch = nullptr;
  RBWS_CHECK(cudaMallocAsync(&scratch, rbws::basis_dot_scratch(n3, count, N), S(stream)));
  cudaError_t e = rbws::basis_dot(n3, count, W, Wstride, N, v, vstride, out,
                                  static_cast<double*>(scratch), S(stream));
  cudaFreeAsync(scratch, S(stream));
  RBWS_CHECK(e);
  return 0;
}

int rbws_expand(int n, int count, const double* W, int64_t Wstride, int N, const double* a,
                double* x, void* stream) {
  if (N < 1) RBWS_FAIL("empty basis");
  RBWS_CHECK(rbws::expand(n, count, W, Wstride, N, a, x, S(stream)));
  return 0;
}

int rbws_deim_step(int n, const double* W, int64_t Wstride, int N, const double* c,
                   const double* v, const uint8_t* excluded, double* col, int64_t* out_idx,
                   double* out_vals, void* stream) {
  void* scratch = nullptr;
  RBWS_CHECK(cudaMallocAsync(&scratch, rbws::deim_scratch_bytes(n), S(stream)));
  cudaError_t e = rbws::deim_step(n, W, Wstride, N, c, v, excluded, col, out_idx, out_vals,
                                  scratch, S(stream));
  cudaFreeAsync(scratch, S(stream));
  RBWS_CHECK(e);
  return 0;
}

int rbws_deim_step_fn(int side, const double* W, int64_t Wstride, int N, const double* c,
                      const double* v, const uint8_t* excluded, double* col, int64_t* out_idx,
                      double* out_vals, void* stream) {
  void* scratch = nullptr;
  RBWS_CHECK(cudaMallocAsync(&scratch, rbws::deim_scratch_bytes(side), S(stream)));
  cudaError_t e = rbws::deim_step(side, W, Wstride, N, c, v, excluded, col, out_idx, out_vals,
                                  scratch, S(stream), false);
  cudaFreeAsync(scratch, S(stream));
  RBWS_CHECK(e);
  return 0;
}

int rbws_dense_solve(int m, const double* A, const double* b, double* x, int* status,
                     void* stream) {
  if (m < 1) RBWS_FAIL("empty system");
  RBWS_CHECK(rbws::dense_solve(m, A, b, x, status, S(stream)));
  return 0;
}

}  // extern "C"

extern "C" {

int rbws_comm_unique_id(uint8_t* out128) {
  if (!out128) RBWS_FAIL("null argument");
  return rbws::comm_unique_id(out128);
}

int rbws_slab_create(rbws_slab** out, rbws_hierarchy* h, int nslabs, int nlocal,
                     const uint8_t* nccl_id, int nprocs, int proc_rank, double omega) {
  if (!out || !h) RBWS_FAIL("null argument");
  if (H(h)->stored) RBWS_FAIL("the slab path takes separable (Kronecker-factor) problems");
  rbws::Comm* comm = nullptr;
  if (nprocs < 1 || proc_rank < 0 || proc_rank >= nprocs) RBWS_FAIL("bad process count / rank");
  if (nprocs > 1 && !nccl_id) RBWS_FAIL("multi-process slabs need an NCCL id");
  // one process with an id: NCCL loopback transport between its own slabs
  if (nccl_id && rbws::comm_create(&comm, nccl_id, nprocs, proc_rank)) return 1;
  rbws::Slab* s = nullptr;
  if (rbws::slab_create(&s, H(h), nslabs, proc_rank * nlocal, nlocal, comm, omega)) {
    delete comm;
    return 1;
  }
  *out = reinterpret_cast<rbws_slab*>(s);
  return 0;
}

int rbws_slab_destroy(rbws_slab* s) {
  delete reinterpret_cast<rbws::Slab*>(s);
  return 0;
}

int rbws_slab_info(const rbws_slab* s, int* first_dist_level, int local, int* k0, int* k1) {
  const rbws::Slab* sl = reinterpret_cast<const rbws::Slab*>(s);
  if (!sl) RBWS_FAIL("null slab");
  if (first_dist_level) *first_dist_level = sl->Ld;
  if (local < 0 || local >= sl->nloc) RBWS_FAIL("local slab index out of range");
  if (k0) *k0 = sl->parts[local].k0[sl->L - 1];
  if (k1) *k1 = sl->parts[local].k1[sl->L - 1];
  return 0;
}

int rbws_slab_setup(rbws_slab* s, const double* theta, int* n_bad, void* stream) {
  if (!s || !theta) RBWS_FAIL("null argument");
  return rbws::slab_setup(reinterpret_cast<rbws::Slab*>(s), theta, n_bad, S(stream));
}

int rbws_slab_load(rbws_slab* s, int which, const double* buf, int64_t p0, int planes,
                   void* stream) {
  if (!s || !buf) RBWS_FAIL("null argument");
  return rbws::slab_load(reinterpret_cast<rbws::Slab*>(s), which ? rbws::SV_F : rbws::SV_X, buf,
                         p0, planes, S(stream));
}

int rbws_slab_store(rbws_slab* s, int which, double* buf, int64_t p0, int planes, void* stream) {
  if (!s || !buf) RBWS_FAIL("null argument");
  return rbws::slab_store(reinterpret_cast<rbws::Slab*>(s), which ? rbws::SV_F : rbws::SV_X, buf,
                          p0, planes, S(stream));
}

int rbws_slab_prolong_x(rbws_slab* s, const double* ec, void* stream) {
  if (!s || !ec) RBWS_FAIL("null argument");
  return rbws::slab_prolong_x(reinterpret_cast<rbws::Slab*>(s), ec, S(stream));
}

int rbws_slab_solve(rbws_slab* s, double delta, int l_max, int* iters, double* hist,
                    double* true_res, int* status, void* stream) {
  if (!s) RBWS_FAIL("null slab");
  return rbws::slab_solve(reinterpret_cast<rbws::Slab*>(s), delta, l_max, iters, hist, true_res,
                          status, S(stream));
}

}  // extern "C"
