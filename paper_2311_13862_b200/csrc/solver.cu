// Batched MGCG runtime (host C++ orchestrating the sm_100a kernels).
//
// Restates, batched over parameter instances:
//   ParametricProblem hierarchy + termwise Galerkin coarsening  (reference grid.py:203-236)
//   mg_context_for: per-mu operators on every level + Cholesky   (multigrid.py:191-202, 154-168)
//   mg_vcycle with damped-Jacobi pre/post sweeps                  (multigrid.py:205-222, kernels.py:98-115)
//   pcg_solve                                                      (krylov.py:42-109)
#include <atomic>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "coarse.cuh"
#include "fine.cuh"
#include "gs.cuh"
#include "solver.cuh"

#include <algorithm>
#include <mutex>

static thread_local std::string g_err;

int rbws_set_error(const char* msg, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s (%s:%d)", msg, file, line);
  g_err = buf;
  return 1;
}

const char* rbws_get_error() { return g_err.c_str(); }

#define RBWS_FAIL(msg) return rbws_set_error(msg, __FILE__, __LINE__)

namespace rbws {

// ---- small device -> host readbacks without the copy engines
// A kernel stores into mapped pinned memory; the stream is synchronised and the
// bytes are memcpy'd to dst.  Control data (active counts, iteration reports)
// must not wait behind a bulk cudaMemcpyAsync queued on a copy engine by
// another stream (the solution download of a pipelined sub-batch).
__global__ void fetch_kernel(const unsigned char* __restrict__ src, unsigned char* dst,
                             int64_t bytes) {
  const int64_t words = bytes / 4;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 3) == 0);
  if (aligned) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
    volatile uint32_t* d4 = reinterpret_cast<volatile uint32_t*>(dst);
    for (int64_t t = t0; t < words; t += stride) d4[t] = s4[t];
    for (int64_t t = words * 4 + t0; t < bytes; t += stride) dst[t] = src[t];
  } else {
    for (int64_t t = t0; t < bytes; t += stride) dst[t] = src[t];
  }
}

cudaError_t fetch_to_host(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  // per-thread staging: host threads driving solves on different streams never wait
  // for each other's synchronisation
  static thread_local unsigned char* stage = nullptr;
  static thread_local size_t cap = 0;
  if (bytes == 0) return cudaSuccess;
  if (bytes > cap) {
    if (stage) cudaFreeHost(stage);
    stage = nullptr;
    cap = std::max<size_t>(bytes, 1 << 16);
    cudaError_t e = cudaHostAlloc((void**)&stage, cap, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) { cap = 0; return e; }
  }
  unsigned char* dstage = nullptr;
  cudaError_t e = cudaHostGetDevicePointer((void**)&dstage, stage, 0);
  if (e != cudaSuccess) return e;
  const int threads = 256;
  const int64_t need = ((int64_t)bytes / 4 + threads - 1) / threads;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, 148));
  count_launch();
  fetch_kernel<<<blocks, threads, 0, stream>>>(static_cast<const unsigned char*>(src), dstage,
                                               (int64_t)bytes);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess) memcpy(dst, stage, bytes);
  return e;
}


static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// the dynamic shared-memory limit is a per-device kernel attribute: remember the largest
// value set for every (kernel, device) pair, under a lock (several host threads may launch)
cudaError_t smem_attr(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{fn, dev}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

template <class T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, count * sizeof(T) + 16);
}

// ------------------------------------------------------------ hierarchy

Hierarchy::~Hierarchy() {
  cudaFree(d_face);
  cudaFree(d_node);
  for (double* p : d_fac) cudaFree(p);
  for (int* p : d_zsame) cudaFree(p);
  for (int* p : d_grp) cudaFree(p);
  cudaFree(d_fzsame);
  for (double* p : d_tcoef) cudaFree(p);
}

// 1D Galerkin product P^T T P of a tridiagonal interior operator
// (diag[i], upper[i] = T(i,i+1)) with linear interpolation nc -> 2nc.
static void galerkin_1d(const double* df, const double* uf, int nf, double* dc, double* uc) {
  const int nc = nf / 2;
  auto T = [&](int i, int j) -> double {
    if (i < 1 || j < 1 || i > nf - 1 || j > nf - 1) return 0.0;
    if (i == j) return df[i];
    if (j == i + 1) return uf[i];
    if (i == j + 1) return uf[j];
    return 0.0;
  };
  auto P = [&](int i, int I) -> double {
    if (i == 2 * I) return 1.0;
    if (i == 2 * I - 1 || i == 2 * I + 1) return 0.5;
    return 0.0;
  };
  for (int I = 0; I <= nc; ++I) { dc[I] = 0.0; uc[I] = 0.0; }
  for (int I = 1; I <= nc - 1; ++I) {
    for (int J = I; J <= I + 1 && J <= nc - 1; ++J) {
      double acc = 0.0;
      for (int i = 2 * I - 1; i <= 2 * I + 1; ++i)
        for (int j = 2 * J - 1; j <= 2 * J + 1; ++j) {
          const double t = T(i, j);
          if (t != 0.0) acc += P(i, I) * t * P(j, J);
        }
      if (J == I) dc[I] = acc; else uc[I] = acc;
    }
  }
}

int kron_factors(int n, int m0, int Q, const double* face, const double* node,
                 std::vector<int>& cells, std::vector<std::vector<double>>& fac) {
  if (Q < 1 || Q > kMaxTerms) RBWS_FAIL("number of affine terms must be in [1, 8]");
  if (m0 < 2) RBWS_FAIL("base grid needs at least 2 cells per dimension");
  if (n % m0) RBWS_FAIL("n must be m0 * 2^J");
  int r = n / m0;
  if (r & (r - 1)) RBWS_FAIL("n must be m0 * 2^J");
  if (r < 2) RBWS_FAIL("need at least 2 levels for coarse-grid correction");
  cells.clear();
  for (int c = m0; c <= n; c *= 2) cells.push_back(c);
  const int L = (int)cells.size();
  fac.assign(L, std::vector<double>());
  {
    const int n1 = n + 1;
    std::vector<double>& f = fac[L - 1];
    f.assign((size_t)Q * 3 * 3 * 2 * n1, 0.0);
    for (int q = 0; q < Q; ++q)
      for (int d = 0; d < 3; ++d)
        for (int a = 0; a < 3; ++a) {
          double* dg = &f[(((size_t)(q * 3 + d) * 3 + a) * 2 + 0) * n1];
          double* up = &f[(((size_t)(q * 3 + d) * 3 + a) * 2 + 1) * n1];
          if (a == d) {
            const double* F = face + (size_t)(q * 3 + d) * n;
            for (int i = 1; i <= n - 1; ++i) dg[i] = F[i - 1] + F[i];
            for (int i = 1; i <= n - 2; ++i) up[i] = -F[i];
          } else {
            const double* N = node + ((size_t)(q * 3 + d) * 3 + a) * n1;
            for (int i = 1; i <= n - 1; ++i) dg[i] = N[i];
          }
        }
  }
  for (int l = L - 2; l >= 0; --l) {
    const int nf = cells[l + 1], nc = cells[l];
    const int nf1 = nf + 1, nc1 = nc + 1;
    std::vector<double>& fc = fac[l];
    const std::vector<double>& ff = fac[l + 1];
    fc.assign((size_t)Q * 3 * 3 * 2 * nc1, 0.0);
    for (int t = 0; t < Q * 3; ++t)
      for (int a = 0; a < 3; ++a)
        galerkin_1d(&ff[((size_t)t * 3 + a) * 2 * nf1], &ff[(((size_t)t * 3 + a) * 2 + 1) * nf1], nf,
                    &fc[((size_t)t * 3 + a) * 2 * nc1], &fc[(((size_t)t * 3 + a) * 2 + 1) * nc1]);
  }
  return 0;
}

int hierarchy_create(Hierarchy** out, int n, int m0, int Q, const double* face,
                     const double* node) {
  if (n < 8) RBWS_FAIL("finest grid must have at least 8 cells");
  if ((m0 - 1) * (m0 - 1) * (m0 - 1) > 125) RBWS_FAIL("coarsest grid too large (m0 <= 6)");
  Hierarchy* h = new Hierarchy();
  h->n = n; h->m0 = m0; h->Q = Q;
  if (kron_factors(n, m0, Q, face, node, h->cells, h->h_fac)) { delete h; return 1; }
  h->levels = (int)h->cells.size();
  const int L = h->levels;
  cudaError_t e = dalloc(&h->d_face, (size_t)Q * 3 * n);
  if (e == cudaSuccess) e = dalloc(&h->d_node, (size_t)Q * 9 * (n + 1));
  if (e == cudaSuccess) e = cudaMemcpy(h->d_face, face, sizeof(double) * Q * 3 * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(h->d_node, node, sizeof(double) * Q * 9 * (n + 1), cudaMemcpyHostToDevice);
  {  // finest level: plane k's z factors (x/y node factors, z faces k-1, k) equal plane k-1's?
    const int n1 = n + 1;
    std::vector<int> fz(n + 1, 0);
    for (int k = 2; k <= n - 1; ++k) {
      int same = 1;
      for (int q = 0; q < Q && same; ++q) {
        const double* F = face + (size_t)q * 3 * n;
        const double* N = node + (size_t)q * 9 * n1;
        same &= N[(0 * 3 + 2) * n1 + k] == N[(0 * 3 + 2) * n1 + k - 1];
        same &= N[(1 * 3 + 2) * n1 + k] == N[(1 * 3 + 2) * n1 + k - 1];
        same &= F[2 * n + k] == F[2 * n + k - 1];
        same &= F[2 * n + k - 1] == F[2 * n + k - 2];
      }
      fz[k] = same;
    }
    h->fine_zchg = 1;  // plane 1
    for (int k = 2; k <= n - 1; ++k) h->fine_zchg += fz[k] ? 0 : 1;
    if (e == cudaSuccess) e = dalloc(&h->d_fzsame, fz.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(h->d_fzsame, fz.data(), sizeof(int) * fz.size(), cudaMemcpyHostToDevice);
  }
  h->d_fac.assign(L, nullptr);
  h->d_zsame.assign(L, nullptr);
  h->d_grp.assign(L, nullptr);
  h->G.assign(L, 0);
  for (int l = 0; l < L && e == cudaSuccess; ++l) {
    e = dalloc(&h->d_fac[l], h->h_fac[l].size());
    if (e == cudaSuccess)
      e = cudaMemcpy(h->d_fac[l], h->h_fac[l].data(), sizeof(double) * h->h_fac[l].size(),
                     cudaMemcpyHostToDevice);
    // per plane k: do all z factors (offsets -1, 0, +1 of every part) equal plane k-1's?
    const int nl = h->cells[l], n1 = nl + 1;
    const std::vector<double>& f = h->h_fac[l];
    std::vector<int> zs(nl + 1, 0);
    auto zt = [&](int t, int k, int o) {
      const double* fz = &f[((size_t)t * 3 + 2) * 2 * n1];
      if (o == 0) return fz[k];
      if (o > 0) return fz[n1 + k];
      return k >= 1 ? fz[n1 + k - 1] : 0.0;
    };
    for (int k = 1; k <= nl; ++k) {
      int same = 1;
      for (int t = 0; t < 3 * Q && same; ++t)
        for (int o = -1; o <= 1; ++o) same &= (zt(t, k, o) == zt(t, k - 1, o)) ? 1 : 0;
      zs[k] = same;
    }
    if (e == cudaSuccess) e = dalloc(&h->d_zsame[l], zs.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(h->d_zsame[l], zs.data(), sizeof(int) * zs.size(), cudaMemcpyHostToDevice);
    // z-groups: terms whose z factors (diagonal and off-diagonal, every plane) are
    // bitwise identical share one z stencil, A = sum_g Z_g (x) (sum_{t in g} theta_t Y_t (x) X_t)
    std::vector<int> grp(3 * Q, -1);
    int G = 0;
    for (int t = 0; t < 3 * Q; ++t) {
      if (grp[t] >= 0) continue;
      grp[t] = G;
      const double* zt0 = &f[((size_t)t * 3 + 2) * 2 * n1];
      for (int t2 = t + 1; t2 < 3 * Q; ++t2)
        if (grp[t2] < 0 &&
            memcmp(zt0, &f[((size_t)t2 * 3 + 2) * 2 * n1], sizeof(double) * 2 * n1) == 0)
          grp[t2] = G;
      ++G;
    }
    h->G[l] = G;
    if (e == cudaSuccess) e = dalloc(&h->d_grp[l], grp.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(h->d_grp[l], grp.data(), sizeof(int) * grp.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) { delete h; RBWS_FAIL(cudaGetErrorString(e)); }
  *out = h;
  return 0;
}

int hierarchy_create_stored(Hierarchy** out, int n, int m0, int Q, const double* coef) {
  if (Q < 1) RBWS_FAIL("need at least one affine term");
  if (m0 < 2) RBWS_FAIL("base grid needs at least 2 cells per dimension");
  if ((m0 - 1) * (m0 - 1) * (m0 - 1) > 125) RBWS_FAIL("coarsest grid too large (m0 <= 6)");
  if (n < 2 * m0 || n % m0) RBWS_FAIL("finest grid must be m0 * 2^J cells with J >= 1");
  {
    const int r = n / m0;
    if (r & (r - 1)) RBWS_FAIL("finest grid must be m0 * 2^J cells");
  }
  Hierarchy* h = new Hierarchy();
  h->n = n; h->m0 = m0; h->Q = Q; h->stored = true;
  for (int c = m0; c <= n; c *= 2) h->cells.push_back(c);
  h->levels = (int)h->cells.size();
  const int L = h->levels;
  h->d_fac.assign(L, nullptr);
  h->d_zsame.assign(L, nullptr);
  h->d_grp.assign(L, nullptr);
  h->G.assign(L, 0);
  h->h_fac.assign(L, {});
  h->d_tcoef.assign(L, nullptr);
  cudaError_t e = cudaSuccess;
  size_t off = 0;
  for (int l = 0; l < L && e == cudaSuccess; ++l) {
    const size_t nl = h->cells[l], cnt = (size_t)Q * 14 * nl * nl * nl;
    e = dalloc(&h->d_tcoef[l], cnt);
    if (e == cudaSuccess)
      e = cudaMemcpy(h->d_tcoef[l], coef + off, sizeof(double) * cnt, cudaMemcpyHostToDevice);
    off += cnt;
  }
  if (e != cudaSuccess) { delete h; RBWS_FAIL(cudaGetErrorString(e)); }
  *out = h;
  return 0;
}

// ------------------------------------------------------------ batch

Batch::~Batch() {
  cudaFree(theta);
  cudaFree(wface);
  for (auto& l : lv) {
    cudaFree(l.b); cudaFree(l.e); cudaFree(l.t1); cudaFree(l.t2); cudaFree(l.t3);
    cudaFree(l.zero); cudaFree(l.dinv); cudaFree(l.u); cudaFree(l.coef);
  }
  cudaFree(L0); cudaFree(d_status);
  cudaFree(r); cudaFree(r2); cudaFree(p); cudaFree(p2); cudaFree(s); cudaFree(t_res);
  cudaFree(rs); cudaFree(alpha); cudaFree(beta); cudaFree(scale);
  cudaFree(active); cudaFree(iters); cudaFree(pstatus); cudaFree(nactive);
  cudaFreeHost(h_nactive);
  cudaFree(partial); cudaFree(partial2); cudaFree(hist);
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  for (cudaEvent_t e : dl_ev) cudaEventDestroy(e);
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  if (gstream) cudaStreamDestroy(gstream);
  for (cudaEvent_t e : gev) if (e) cudaEventDestroy(e);
}

Sep7 Batch::fine_op() const {
  Sep7 op;
  op.n = h->n; op.Q = h->Q; op.face = h->d_face; op.node = h->d_node; op.theta = theta;
  op.zchg = h->fine_zchg;
  op.fz = h->d_fzsame;
  op.wface = wface;
  op.wstride = wstride;
  return op;
}

static bool fem_shared(const Hierarchy* h) {
  static const char* env = getenv("RBWS_FEM_SHARED");
  return h->Q <= 4 && !(env && atoi(env) == 0);
}

int batch_create(Batch** out, Hierarchy* h, int cap, int nu, double omega, int maxl) {
  if (cap < 1) RBWS_FAIL("batch capacity must be positive");
  if (nu < 0) RBWS_FAIL("smoothing count must be non-negative");
  if (nu == 0) RBWS_FAIL("nu = 0 (no smoothing) is not supported by the batched V-cycle");
  Batch* b = new Batch();
  b->h = h; b->cap = cap; b->nu = nu; b->omega = omega;
  {
    const char* g = getenv("RBWS_GRAPH");
    b->use_graph = g ? atoi(g) != 0 : b->use_graph;
    const char* fr = getenv("RBWS_FUSED_RESTRICT");  // "0": separate pre-smoothing + restriction
    b->fuse_restrict = fr ? atoi(fr) != 0 : true;
  }
  const int L = h->levels;
  b->maxl = (maxl <= 0 || maxl > L) ? L : maxl;
  cudaError_t e = dalloc(&b->theta, (size_t)cap * h->Q);
  b->lv.resize(L);
  for (int l = 0; l < b->maxl && e == cudaSuccess; ++l) {
    LevelBuf& lb = b->lv[l];
    lb.n = h->cells[l];
    const size_t V = (size_t)vec_doubles(lb.n, cap);
    const size_t n3 = (size_t)lb.n * lb.n * lb.n;
    auto zalloc = [&](double** p, size_t cnt) {
      if (e != cudaSuccess) return;
      e = dalloc(p, cnt);
      if (e == cudaSuccess) e = cudaMemset(*p, 0, cnt * sizeof(double));
    };
    zalloc(&lb.t1, V);
    zalloc(&lb.dinv, V);
    if (nu != 1) { zalloc(&lb.t2, V); zalloc(&lb.t3, V); zalloc(&lb.zero, V); }
    if (l >= 1 && (l < L - 1 || h->stored)) zalloc(&lb.u, V);
    // stored-coefficient hierarchies: per-instance coefficients on the coarse levels; the
    // finest level combines the batch-shared term coefficients on the fly (Q <= 4, unless
    // RBWS_FEM_SHARED=0) and keeps no per-instance copy
    if (e == cudaSuccess && h->stored && (l < L - 1 || !fem_shared(h)))
      e = dalloc(&lb.coef, (size_t)14 * cap * n3);
    // levels whose terms fall into more z-groups than the grouped Kronecker kernel takes:
    // stored per-instance coefficients (without the memory, the matrix-free 27-coefficient
    // kernel runs instead)
    if (e == cudaSuccess && !h->stored && l >= 1 && l < L - 1 && h->G[l] > kCoarseMaxGroups) {
      if (dalloc(&lb.coef, (size_t)14 * cap * n3) != cudaSuccess) {
        (void)cudaGetLastError();
        lb.coef = nullptr;
      }
    }
    if (l < L - 1) {
      zalloc(&lb.b, V);
      zalloc(&lb.e, V);
      (void)n3;
    }
  }
  if (e == cudaSuccess) {
    const int m1 = h->m0 - 1, m = m1 * m1 * m1;
    e = dalloc(&b->L0, (size_t)cap * m * m);
  }
  const size_t VF = (size_t)vec_doubles(h->n, cap);
  if (e == cudaSuccess) e = dalloc(&b->d_status, cap);
  // coefficients whose z factors change on most planes: stored face weights (SCW kernels);
  // without the memory the register-refresh kernels run instead
  const char* scw_env = getenv("RBWS_SCW");  // "0": keep the register-refresh kernels
  const bool scw = !(scw_env && atoi(scw_env) == 0);
  if (e == cudaSuccess && scw && b->maxl == L && h->fine_zchg >= kFineStoredWeightsMinChanges) {
    b->wstride = (int64_t)VF;
    if (dalloc(&b->wface, (size_t)3 * VF) != cudaSuccess) {
      (void)cudaGetLastError();
      b->wface = nullptr;
    } else {
      e = cudaMemset(b->wface, 0, sizeof(double) * 3 * VF);
    }
  }
  for (double** pp : {&b->r, &b->p, &b->p2, &b->s, &b->t_res}) {
    if (b->maxl < L) break;  // coarse levels only (slab path): no finest-level PCG vectors
    if (e == cudaSuccess) e = dalloc(pp, VF);
    if (e == cudaSuccess) e = cudaMemset(*pp, 0, VF * sizeof(double));
  }
  for (double** pp : {&b->rs, &b->alpha, &b->beta, &b->scale})
    if (e == cudaSuccess) e = dalloc(pp, cap);
  for (int** pp : {&b->active, &b->iters, &b->pstatus})
    if (e == cudaSuccess) e = dalloc(pp, cap);
  if (e == cudaSuccess) e = dalloc(&b->nactive, 1);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&b->h_nactive, sizeof(int));
  if (e == cudaSuccess) {
    int64_t t = sep7_geom(h->n, 1).tiles;
    for (int c = 2; c <= cap; c *= 2) t = std::max<int64_t>(t, sep7_geom(h->n, c).tiles);
    t = std::max<int64_t>(t, sep7_geom(h->n, cap).tiles);
    t = std::max<int64_t>(t, vec_tiles(h->n));
    for (int c = 1; c <= cap; c *= 2)
      t = std::max<int64_t>(t, std::max(fine_geom(h->n, c).tiles, fine_post_tiles(h->n, c)));
    t = std::max<int64_t>(t, std::max(fine_geom(h->n, cap).tiles, fine_post_tiles(h->n, cap)));
    b->partial_cap = t;
    e = dalloc(&b->partial, (size_t)cap * t);
    if (e == cudaSuccess) e = dalloc(&b->partial2, (size_t)cap * t);
  }
  if (e != cudaSuccess) { delete b; RBWS_FAIL(cudaGetErrorString(e)); }
  *out = b;
  return 0;
}

void Batch::drop_graph() {
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  gexec = nullptr;
  graph = nullptr;
  gkey_x = nullptr;
  gkey_active = nullptr;
}

int batch_set_smoother(Batch* b, int kind) {
  if (kind != 0 && kind != 1) RBWS_FAIL("smoother kind must be 0 (jacobi) or 1 (gauss-seidel)");
  Hierarchy* h = b->h;
  const int L = h->levels;
  if (kind == 1) {
    if (b->maxl < L) RBWS_FAIL("Gauss-Seidel needs the finest level");
    const size_t VF = (size_t)vec_doubles(h->n, b->cap);
    cudaError_t e = cudaSuccess;
    if (!b->wface && !h->stored) {
      b->wstride = (int64_t)VF;
      e = dalloc(&b->wface, 3 * VF);
      if (e == cudaSuccess) e = cudaMemset(b->wface, 0, sizeof(double) * 3 * VF);
    }
    for (int l = 1; l < (h->stored ? L : L - 1) && e == cudaSuccess; ++l) {
      LevelBuf& lb = b->lv[l];
      if (lb.coef) continue;
      const size_t n3 = (size_t)lb.n * lb.n * lb.n;
      e = dalloc(&lb.coef, (size_t)14 * b->cap * n3);
    }
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  }
  if (kind != b->smoother) b->drop_graph();  // the captured V-cycle used the old smoother
  b->smoother = kind;
  b->count = 0;  // set up again
  return 0;
}

int batch_setup(Batch* b, const double* theta, int count, cudaStream_t stream) {
  if (count < 1 || count > b->cap) RBWS_FAIL("batch count outside [1, capacity]");
  Hierarchy* h = b->h;
  b->count = count;
  cudaError_t e = cudaMemcpyAsync(b->theta, theta, sizeof(double) * count * h->Q,
                                  cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  const int L = h->levels;
  LaunchCtx lc{stream, nullptr};
  if (h->stored) {  // assembled problem: per-instance coefficients on every level, dense coarsest
    for (int l = 0; l < b->maxl && e == cudaSuccess; ++l)
      e = stored_combine(h->cells[l], h->Q, h->d_tcoef[l], b->theta, count, b->lv[l].coef,
                         b->lv[l].dinv, stream);
    if (e == cudaSuccess)
      e = coarse_factor_stored(h->m0, h->Q, h->d_tcoef[0], b->theta, count, b->L0, b->d_status,
                               stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    return 0;
  }
  // fine level 1/diag (and the stored face weights of the SCW kernels)
  if (b->maxl == L) e = fine_dinv(b->fine_op(), count, h->d_fzsame, b->lv[L - 1].dinv, stream);
  if (e == cudaSuccess && b->wface) e = fine_faces(b->fine_op(), count, b->wface, b->wstride, stream);
  // coarse levels are matrix-free (Kronecker factors): only 1/diag is stored
  for (int l = 1; l < std::min(L - 1, b->maxl) && e == cudaSuccess; ++l)
    e = b->lv[l].coef
            ? coarse_build_coef(h->coarse_op(l), b->theta, count, b->lv[l].coef, b->lv[l].dinv,
                                stream)
            : coarse_launch(4, h->coarse_op(l), b->theta, count,
                      nullptr, nullptr, b->lv[l].dinv, 0.0, lc);
  if (e == cudaSuccess)
    e = coarse_factor_kf(h->m0, h->Q, h->d_fac[0], b->theta, count, b->L0, b->d_status, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  return 0;
}

int Batch::prof_begin(cudaStream_t s) {
  if (ev_used + 2 > ev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
  }
  const int idx = (int)ev_used++;
  cudaEventRecord(ev[idx], s);
  return idx;
}

void Batch::prof_end(int cls, int start, cudaStream_t s) {
  const int idx = (int)ev_used++;
  cudaEventRecord(ev[idx], s);
  recs.push_back({cls, start, idx, cur_active});
}

void Batch::prof_flush() {
  static const bool dump = getenv("RBWS_PROF_DUMP") != nullptr;  // per-launch trace (stderr)
  for (auto& r : recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev[r[1]], ev[r[2]]) == cudaSuccess) {
      if (dump) fprintf(stderr, "PROF %d %d %.4f\n", r[0], r[3], ms);
      prof_ms[r[0]] += ms;
      prof_calls[r[0]] += 1;
      prof_units[r[0]] += r[3];
    }
  }
  recs.clear();
  ev_used = 0;
}

// The fused coarse tail (tail.cu) is opt-in (rbws_set_kernel_variant(2, 1) or RBWS_TAIL=1):
// bitwise the per-level kernels, 13 -> 5 launches per V-cycle below the 32^3 level, but on
// configs[1] its one CTA per instance (phases separated by CTA barriers, 16 warps per SM) takes
// 0.29 ms per full batch against 0.23 ms for the per-level kernels, and the step is unchanged
// (13.9-14.0k solves/s either way; it wins only on short batches)
static std::atomic<int> g_tail{[] {
  const char* e = getenv("RBWS_TAIL");
  return (e && atoi(e) == 1) ? 1 : 0;
}()};
int solver_set_tail(int v) {
  if (v < -1 || v > 1) return 1;
  g_tail.store(v == 1 ? 1 : 0);
  return 0;
}
static int variant_key() {
  return fine_variant() + 1024 * g_tail.load() + 2048 * fine_cgp_variant();
}

// the fused coarse tail (tail.cu) serves level lvl and everything below it?
bool Batch::tail_level(int lvl, const LaunchCtx& lc) const {
  if (!g_tail.load(std::memory_order_relaxed) || h->stored || smoother != 0 || nu != 1)
    return false;
  if (lvl < 1 || lvl >= h->levels - 1 || lvl > kTailMaxLevels || lc.zhi > 0) return false;
  if (h->cells[lvl] > 16 || (lvl + 1 < h->levels - 1 && h->cells[lvl + 1] <= 16)) return false;
  TailArgs t;
  t.LT = lvl;
  for (int l = 0; l <= lvl; ++l) {
    t.n[l] = h->cells[l];
    if (l >= 1 && (h->G[l] != h->G[lvl] || lv[l].coef || !lv[l].u)) return false;
  }
  return coarse_tail_fits(t, h->G[lvl]);
}

// one V-cycle for A^lvl out = b from zero, per active instance
int Batch::vcycle(int lvl, const double* bb, double* out, double* dot_partial,
                  const LaunchCtx& lc) {
  cudaError_t e = cudaSuccess;
  if (lvl == 0) {
    e = coarse_solve(h->m0, count, L0, bb, out, lc);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    return 0;
  }
  if (tail_level(lvl, lc)) {  // levels <= 16 cells and the coarsest solve in one kernel
    TailArgs t;
    t.LT = lvl;
    t.Q = h->Q;
    for (int l = 0; l <= lvl; ++l) {
      t.n[l] = h->cells[l];
      t.fac[l] = h->d_fac[l];
      t.grp[l] = h->d_grp[l];
    }
    t.theta = theta;
    t.b = bb;
    t.u = lv[lvl].u;
    t.e = out;
    t.L0 = L0;
    t.active = lc.active;
    t.omega = omega;
    e = coarse_tail_launch(t, h->G[lvl], count, lc.stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    return 0;
  }
  const bool fine = h->sep_fine(lvl);
  // top level of a stored-coefficient hierarchy: coarse-type kernels, the PCG dot separately
  const bool stop = h->stored && lvl == h->levels - 1;
  LevelBuf& l = lv[lvl];
  LevelBuf& c = lv[lvl - 1];
  const int n = l.n;
  auto op = [&](int mode, int dot, const double* x, const double* rhs, double* y,
                double* part) -> cudaError_t {
    if (fine) {
      const Sep7 fo = fine_op();
      if (mode == MODE_PRE) return fine_pre(fo, count, rhs, l.dinv, y, omega, lc);
      if (mode == MODE_JACOBI)
        return fine_jacobi(fo, count, x, rhs, y, omega, dot == DOT_NONE ? nullptr : part, lc);
      if (mode == MODE_RESID) return fine_resid(fo, count, x, rhs, y, nullptr, lc);
      return sep7_launch(fo, count, mode, dot, x, rhs, l.dinv, y, part, omega, lc);
    }
    // coarse levels: the pre-smoothing residual is a residual of the pre-scaled rhs l.u
    if (mode == MODE_PRE)
      return coarse_launch(1, cop(lvl), theta, count, l.u, rhs, y,
                           omega, lc);
    const int cm = (mode == MODE_JACOBI) ? 2 : (mode == MODE_RESID) ? 1 : 0;
    return coarse_launch(cm, cop(lvl), theta, count, x, rhs, y,
                         omega, lc);
  };
  const int fdot = (fine && dot_partial) ? DOT_BY : DOT_NONE;
  const bool pf = fine && prof_on;
  if (smoother == 1) {  // Gauss-Seidel: forward sweeps from zero, backward after correction
    const int64_t n3 = (int64_t)n * n * n;
    auto gs = [&](bool fwd) -> cudaError_t {
      return fine ? gs7_sweep(n, count, wface, wstride, bb, out, fwd, lc)
                  : gs27_sweep(n, count, l.coef, bb, out, fwd, lc);
    };
    e = cudaMemsetAsync(out, 0, sizeof(double) * count * n3, lc.stream);
    for (int s = 0; s < nu && e == cudaSuccess; ++s) e = gs(true);
    if (e == cudaSuccess) e = op(MODE_RESID, DOT_NONE, out, bb, l.t1, nullptr);
    if (e == cudaSuccess) e = restrict_launch(n, count, l.t1, c.b, lc);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    if (vcycle(lvl - 1, c.b, c.e, nullptr, lc)) return 1;
    e = prolong_launch(n, count, 0, c.e, out, nullptr, nullptr, 0.0, lc);
    for (int s = 0; s < nu && e == cudaSuccess; ++s) e = gs(false);
    if (e == cudaSuccess && (fine || stop) && dot_partial)
      e = vec_dot(n, count, bb, n3, out, n3, dot_partial, lc);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    return 0;
  }
  if (nu == 1) {
    int t0 = pf ? prof_begin(lc.stream) : -1;
    // finest level, whole instances per CTA: the pre-smoothing kernel also runs the x and z
    // passes of the restriction (r1 never reaches HBM), a light kernel the y pass
    const bool fused = fine && fuse_restrict && lvl - 1 >= 1 && fine_pre_xz_ok(fine_op(), count, lc);
    if (fine) {  // (the coarse levels of the recursion leave these alone)
      fused_used = fused;
      sw_used = fine_pre_scaled(fine_op());
    }
    if (stop) e = vec_scale_dinv(n, count, omega, l.dinv, bb, l.u, lc.stream);
    if (e == cudaSuccess && !(fine && fused && pre_done))  // (pre_done: l.t1 holds t already)
      e = fused ? fine_pre_xz(fine_op(), count, bb, l.dinv, l.t1, omega, lc)
                : op(MODE_PRE, DOT_NONE, nullptr, bb, l.t1, nullptr);
    // (pre_done: nothing was launched for the pre-smoothing class)
    if (pf && !(fine && fused && pre_done)) {
      prof_end(PROF_FINE_PRE, t0, lc.stream);
      t0 = prof_begin(lc.stream);
    }
    // the restriction also writes the next level's pre-scaled rhs u = w D^-1 b
    if (e == cudaSuccess)
      e = fused ? restrict_y_launch(n, count, l.t1, c.b, lc, c.dinv, c.u, omega)
          : (lvl - 1 >= 1) ? restrict_launch(n, count, l.t1, c.b, lc, c.dinv, c.u, omega)
                           : restrict_launch(n, count, l.t1, c.b, lc);
    if (pf) { prof_end(PROF_FINE_RESTRICT, t0, lc.stream); t0 = prof_begin(lc.stream); }
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    if (vcycle(lvl - 1, c.b, c.e, nullptr, lc)) return 1;
    if (pf) { prof_end(PROF_COARSE, t0, lc.stream); t0 = prof_begin(lc.stream); }
    if (fine) {  // prolongation fused into the post-smoothing sweep
      e = fine_post_prolong(fine_op(), count, bb, l.dinv, c.e, out, omega,
                            fdot == DOT_NONE ? nullptr : dot_partial, lc);
      if (pf) prof_end(PROF_FINE_POST, t0, lc.stream);
    } else {
      e = prolong_launch(n, count, 2, c.e, l.t1, l.u, nullptr, omega, lc);
      if (e == cudaSuccess) e = op(MODE_JACOBI, fdot, l.t1, bb, out, dot_partial);
      if (e == cudaSuccess && stop && dot_partial)
        e = vec_dot(n, count, bb, (int64_t)n * n * n, out, (int64_t)n * n * n, dot_partial, lc);
    }
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    return 0;
  }
  // generic nu: u in t1/t2 ping-pong, residual in t3
  double* u = l.zero;
  double* bufs[2] = {l.t1, l.t2};
  int nb = 0;
  for (int s = 0; s < nu && e == cudaSuccess; ++s) {
    e = op(MODE_JACOBI, DOT_NONE, u, bb, bufs[nb], nullptr);
    u = bufs[nb];
    nb ^= 1;
  }
  if (e == cudaSuccess) e = op(MODE_RESID, DOT_NONE, u, bb, l.t3, nullptr);
  if (e == cudaSuccess) e = restrict_launch(n, count, l.t3, c.b, lc);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  if (vcycle(lvl - 1, c.b, c.e, nullptr, lc)) return 1;
  e = prolong_launch(n, count, 0, c.e, u, nullptr, nullptr, 0.0, lc);
  for (int s = 0; s < nu && e == cudaSuccess; ++s) {
    const bool last = (s == nu - 1);
    double* dst = last ? out : (u == l.t1 ? l.t2 : l.t1);
    e = op(MODE_JACOBI, last ? fdot : DOT_NONE, u, bb, dst, last ? dot_partial : nullptr);
    u = dst;
  }
  if (e == cudaSuccess && stop && dot_partial)
    e = vec_dot(n, count, bb, (int64_t)n * n * n, out, (int64_t)n * n * n, dot_partial, lc);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  return 0;
}

// ------------------------------------------------------------ PCG scalars

// one warp per instance: deterministic sum of `tiles` partials
__device__ __forceinline__ double warp_sum_partials(const double* part, int tiles) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int t = lane; t < tiles; t += 32) s += part[t];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  return __shfl_sync(0xffffffffu, s, 0);
}

#define WARP_MU                                                       \
  const int mu = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); \
  const int lane = threadIdx.x & 31;                                  \
  if (mu >= count) return;

__global__ void pcg_init_kernel(int count, const double* pf, int ftiles, int fshared,
                                const double* prr, int tiles, double delta, int l_max,
                                double* scale, double* hist, int hist_len, int* active,
                                int* iters, int* status, int* nactive) {
  WARP_MU
  const double ff = warp_sum_partials(pf + (fshared ? 0 : (int64_t)mu * ftiles), ftiles);
  const double rr = warp_sum_partials(prr + (int64_t)mu * tiles, tiles);
  if (lane == 0) {
    const double fn = sqrt(ff);
    const double sc = (fn == 0.0) ? 1.0 : fn;
    scale[mu] = sc;
    const double h0 = sqrt(rr) / sc;
    double* H = hist + (int64_t)mu * hist_len;
    H[0] = h0;
    for (int k = 1; k < hist_len; ++k) H[k] = nan("");
    iters[mu] = 0;
    status[mu] = (fn == 0.0) ? 4 : 0;  // bit 2: absolute norms
    const int a = (h0 > delta && l_max > 0) ? 1 : 0;
    active[mu] = a;
    if (a) atomicAdd(nactive, 1);
  }
}

__global__ void pcg_rs_kernel(int count, const double* prs, int tiles, double* rs,
                              const int* active) {
  WARP_MU
  if (!active[mu]) return;
  const double v = warp_sum_partials(prs + (int64_t)mu * tiles, tiles);
  if (lane == 0) rs[mu] = v;
}

__global__ void pcg_alpha_kernel(int count, const double* ppap, int tiles, const double* rs,
                                 double* alpha, int* active, int* status) {
  WARP_MU
  if (!active[mu]) return;
  const double pap = warp_sum_partials(ppap + (int64_t)mu * tiles, tiles);
  if (lane == 0) {
    if (!(pap > 0.0)) {
      status[mu] |= 1;  // non-positive curvature: operator not SPD
      active[mu] = 0;
      alpha[mu] = 0.0;
    } else {
      alpha[mu] = rs[mu] / pap;
    }
  }
}

__global__ void pcg_check_kernel(int count, const double* prr, int tiles, const double* scale,
                                 double delta, int l_max, double* hist, int hist_len,
                                 int* active, int* iters, int* nactive) {
  WARP_MU
  if (!active[mu]) return;
  const double rr = warp_sum_partials(prr + (int64_t)mu * tiles, tiles);
  if (lane == 0) {
    const double rel = sqrt(rr) / scale[mu];
    const int k = iters[mu] + 1;
    iters[mu] = k;
    hist[(int64_t)mu * hist_len + k] = rel;
    if (rel <= delta || k >= l_max) active[mu] = 0;
    else atomicAdd(nactive, 1);
  }
}

__global__ void pcg_beta_kernel(int count, const double* prs, int tiles, double* rs,
                                double* beta, const int* active) {
  WARP_MU
  if (!active[mu]) return;
  const double v = warp_sum_partials(prs + (int64_t)mu * tiles, tiles);
  if (lane == 0) {
    beta[mu] = v / rs[mu];
    rs[mu] = v;
  }
}

__global__ void pcg_true_kernel(int count, const double* prr, int tiles, const double* scale,
                                double* out) {
  WARP_MU
  const double rr = warp_sum_partials(prr + (int64_t)mu * tiles, tiles);
  if (lane == 0) out[mu] = sqrt(rr) / scale[mu];
}

static inline dim3 warp_grid(int count) { return dim3((count + 7) / 8); }

// host launchers of the per-instance PCG scalar kernels (shared with slab.cu)
cudaError_t pcg_init(int count, const double* pf, int ftiles, int fshared, const double* prr,
                     int tiles, double delta, int l_max, double* scale, double* hist,
                     int hist_len, int* active, int* iters, int* status, int* nactive,
                     cudaStream_t s) {
  count_launch();
  pcg_init_kernel<<<warp_grid(count), 256, 0, s>>>(count, pf, ftiles, fshared, prr, tiles, delta,
                                                   l_max, scale, hist, hist_len, active, iters,
                                                   status, nactive);
  return cudaGetLastError();
}
cudaError_t pcg_rs(int count, const double* prs, int tiles, double* rs, const int* active,
                   cudaStream_t s) {
  count_launch();
  pcg_rs_kernel<<<warp_grid(count), 256, 0, s>>>(count, prs, tiles, rs, active);
  return cudaGetLastError();
}
cudaError_t pcg_alpha(int count, const double* ppap, int tiles, const double* rs, double* alpha,
                      int* active, int* status, cudaStream_t s) {
  count_launch();
  pcg_alpha_kernel<<<warp_grid(count), 256, 0, s>>>(count, ppap, tiles, rs, alpha, active, status);
  return cudaGetLastError();
}
cudaError_t pcg_check(int count, const double* prr, int tiles, const double* scale, double delta,
                      int l_max, double* hist, int hist_len, int* active, int* iters,
                      int* nactive, cudaStream_t s) {
  count_launch();
  pcg_check_kernel<<<warp_grid(count), 256, 0, s>>>(count, prr, tiles, scale, delta, l_max, hist,
                                                    hist_len, active, iters, nactive);
  return cudaGetLastError();
}
cudaError_t pcg_beta(int count, const double* prs, int tiles, double* rs, double* beta,
                     const int* active, cudaStream_t s) {
  count_launch();
  pcg_beta_kernel<<<warp_grid(count), 256, 0, s>>>(count, prs, tiles, rs, beta, active);
  return cudaGetLastError();
}
cudaError_t pcg_true(int count, const double* prr, int tiles, const double* scale, double* out,
                     cudaStream_t s) {
  count_launch();
  pcg_true_kernel<<<warp_grid(count), 256, 0, s>>>(count, prr, tiles, scale, out);
  return cudaGetLastError();
}

// Streaming download: copy the solutions of instances that stopped iterating since the
// last call (all remaining ones when `all`) to the host on out.copy_stream, after the
// compute stream reaches this point.  Consecutive instances go in one copy.
// Two phases, so that the host does not hold back the next iteration's launches while it
// enqueues up to `count` copies (3-5 us of host time each): dl_mark reads the active flags,
// claims the finished instances and records the compute-stream event their x is final at;
// dl_flush enqueues the claimed copies behind that event.  The PCG loops call dl_mark where an
// iteration's active count is known and dl_flush after the next iteration's kernels are
// launched (x of a stopped instance is never written again).
static int dl_mark(Batch* b, const PcgOut& out, int call, bool all, cudaStream_t stream) {
  if (!out.x_host) return 0;
  const int count = b->count;
  if (!all) {
    cudaError_t e = fetch_to_host(b->h_active.data(), b->active, sizeof(int) * count, stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  }
  bool any = false;
  for (int m = 0; m < count; ++m)
    if (!b->h_sent[m] && (all || !b->h_active[m])) {
      b->h_sent[m] = 2;  // claimed, copy not enqueued yet
      any = true;
    }
  if (!any) return 0;
  while ((size_t)call >= b->dl_ev.size()) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    b->dl_ev.push_back(ev);
  }
  cudaError_t e = cudaEventRecord(b->dl_ev[call], stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  b->dl_pending.push_back(call);
  return 0;
}

static int dl_flush(Batch* b, const double* x, const PcgOut& out) {
  if (!out.x_host || b->dl_pending.empty()) return 0;
  const int count = b->count;
  const int64_t n3 = (int64_t)b->h->n * b->h->n * b->h->n;
  cudaError_t e = cudaSuccess;
  // the claimed instances' x became final no later than the last recorded event
  e = cudaStreamWaitEvent(out.copy_stream, b->dl_ev[b->dl_pending.back()], 0);
  b->dl_pending.clear();
  int m = 0;
  while (m < count && e == cudaSuccess) {
    if (b->h_sent[m] != 2) { ++m; continue; }
    int m1 = m;
    while (m1 < count && b->h_sent[m1] == 2 && (out.host_stride == n3 || m1 == m)) {
      b->h_sent[m1] = 1;
      ++m1;
    }
    e = cudaMemcpyAsync(out.x_host + (int64_t)m * out.host_stride, x + (int64_t)m * n3,
                        sizeof(double) * n3 * (m1 - m), cudaMemcpyDeviceToHost, out.copy_stream);
    m = m1;
  }
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  return 0;
}

// mark + flush in one step (the end of a solve, instances converged at x0)
static int stream_download(Batch* b, const double* x, const PcgOut& out, int call, bool all,
                           cudaStream_t stream) {
  if (dl_mark(b, out, call, all, stream)) return 1;
  return dl_flush(b, x, out);
}

// the CG update may carry the next V-cycle's pre-smoothing residual + x/z restriction (cgp.cu)
static bool cgp_ok(Batch* b, const Sep7& op, const LaunchCtx& lc) {
  const int L = b->h->levels;
  return b->nu == 1 && b->smoother == 0 && b->fuse_restrict && L - 2 >= 1 &&
         fine_cgp_ok(op, b->count, lc) && fine_pre_xz_ok(op, b->count, lc);
}

// device-side loop condition: keep iterating while any instance is active
__global__ void pcg_cond_kernel(cudaGraphConditionalHandle h, const int* nactive) {
  cudaGraphSetConditional(h, *nactive > 0 ? 1u : 0u);
}

// PCG iterations 1.. as one CUDA graph: a WHILE conditional node whose body (two
// iterations, so the search-direction buffers alternate back) is captured from the same
// launches the host loop issues; the condition is set on the device from the active
// count, so no host synchronisation happens between iterations.
static int pcg_graph_run(Batch* b, const Sep7& op, double* x, int tiles, int vtiles,
                         double delta, int l_max, int hl, const LaunchCtx& act_in,
                         cudaStream_t user) {
  const int count = b->count, L = b->h->levels;
  // the legacy default stream cannot be captured: capture and launch on a private stream
  // ordered after / before the caller's
  cudaStream_t stream = user;
  if (user == nullptr || user == cudaStreamLegacy) {
    if (!b->gstream) {
      cudaError_t e0 = cudaStreamCreateWithFlags(&b->gstream, cudaStreamNonBlocking);
      if (e0 == cudaSuccess) e0 = cudaEventCreateWithFlags(&b->gev[0], cudaEventDisableTiming);
      if (e0 == cudaSuccess) e0 = cudaEventCreateWithFlags(&b->gev[1], cudaEventDisableTiming);
      if (e0 != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e0));
    }
    stream = b->gstream;
    cudaError_t e0 = cudaEventRecord(b->gev[0], user);
    if (e0 == cudaSuccess) e0 = cudaStreamWaitEvent(stream, b->gev[0], 0);
    if (e0 != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e0));
  }
  LaunchCtx act = act_in;
  act.stream = stream;
  const bool hit = b->gexec && b->gkey_x == x && b->gkey_count == count &&
                   b->gkey_delta == delta && b->gkey_lmax == l_max && b->gkey_hl == hl &&
                   b->gkey_active == act.active && b->gkey_smoother == b->smoother &&
                   b->gkey_fused == (int)b->fuse_restrict && b->gkey_wface == b->wface &&
                   b->gkey_rcur == b->rcur &&
                   b->gkey_variant == variant_key();
  cudaError_t e = cudaSuccess;
  if (!hit) {
    b->drop_graph();
    cudaGraph_t g;
    e = cudaGraphCreate(&g, 0);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    b->graph = g;
    cudaGraphConditionalHandle hnd;
    e = cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hnd;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const int64_t c0 = launch_count();
    e = cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    int rc = 0;
    for (int half = 0; half < 2 && !rc && e == cudaSuccess; ++half) {
      double* p_old = half ? b->p2 : b->p;
      double* p_new = half ? b->p : b->p2;
      e = fine_papply(op, count, b->s, p_old, b->beta, p_new, b->partial, act);
      if (e != cudaSuccess) break;
      count_launch();
      pcg_alpha_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->rs,
                                                             b->alpha, b->active, b->pstatus);
      const bool cgp = cgp_ok(b, op, act);
      if (cgp) {  // (out of place: two halves bring the residual back to the buffer it started in)
        double* r_out = (b->rcur == b->r) ? b->r2 : b->r;
        e = fine_cg_update_pre(op, count, p_new, x, b->rcur, r_out, b->alpha, b->partial,
                               b->lv[L - 1].t1, b->omega, act);
        b->rcur = r_out;
      } else {
        e = fine_cg_update(op, count, p_new, x, b->rcur, b->alpha, b->partial, act);
      }
      if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
      if (e != cudaSuccess) break;
      count_launch();
      pcg_check_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->scale,
                                                             delta, l_max, b->hist, hl, b->active,
                                                             b->iters, b->nactive);
      b->pre_done = cgp;
      rc = b->vcycle(L - 1, b->rcur, b->s, b->partial, act);
      b->pre_done = false;
      if (rc) break;
      count_launch();
      pcg_beta_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, vtiles, b->rs,
                                                            b->beta, b->active);
    }
    if (!rc && e == cudaSuccess) {
      count_launch();
      pcg_cond_kernel<<<1, 1, 0, stream>>>(hnd, b->nactive);
      e = cudaGetLastError();
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(stream, &captured);
    if (rc) return 1;
    if (e == cudaSuccess) e = ec;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&b->gexec, g, 0);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    b->gbody_launches = launch_count() - c0;
    count_launches(-b->gbody_launches);  // captured, not executed
    b->gkey_x = x; b->gkey_count = count; b->gkey_delta = delta; b->gkey_lmax = l_max;
    b->gkey_hl = hl; b->gkey_active = act.active; b->gkey_smoother = b->smoother;
    b->gkey_fused = (int)b->fuse_restrict; b->gkey_wface = b->wface;
    b->gkey_rcur = b->rcur;
    b->gkey_variant = variant_key();
  }
  e = cudaGraphLaunch(b->gexec, stream);
  if (e == cudaSuccess && stream != user) {
    e = cudaEventRecord(b->gev[1], stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, b->gev[1], 0);
  }
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  return 0;
}

// ------------------------------------------------------------ PCG on a stored-coefficient
// hierarchy (assembled FEM problems): the reference loop (krylov.py:73-101) over generic
// kernels — 27-point apply, elementwise updates, deterministic per-instance dot partials

__global__ void __launch_bounds__(256) pcg_xpby_kernel(int64_t n3, const double* __restrict__ s,
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

__global__ void __launch_bounds__(256) pcg_update_kernel(int64_t n3, const double* __restrict__ p,
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

static int pcg_solve_stored(Batch* b, const double* f, int64_t f_stride, double* x, double delta,
                            int l_max, const PcgOut& out, cudaStream_t stream) {
  Hierarchy* h = b->h;
  const int count = b->count, n = h->n, L = h->levels;
  const int64_t n3 = (int64_t)n * n * n;
  if (f_stride == 0 && count > 1)
    RBWS_FAIL("stored-coefficient problems take one rhs per instance (f_stride = n^3)");
  const int hl = b->hist_len;
  const int tiles = vec_tiles(n);
  const CoarseOp op = b->cop(L - 1);
  LaunchCtx all{stream, nullptr};
  LaunchCtx act{stream, b->active};
  const dim3 vg((unsigned)((n3 + 255) / 256), count);
  cudaError_t e = vec_dot(n, count, f, n3, f, n3, b->partial2, all);
  if (e == cudaSuccess) e = coarse_launch(1, op, b->theta, count, x, f, b->r, 0.0, all);
  if (e == cudaSuccess) e = vec_dot(n, count, b->r, n3, b->r, n3, b->partial, all);
  if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  count_launch();
  pcg_init_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial2, tiles, 0, b->partial,
                                                        tiles, delta, l_max, b->scale, b->hist,
                                                        hl, b->active, b->iters, b->pstatus,
                                                        b->nactive);
  e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  b->cur_active = *b->h_nactive;
  int dl_call = 0;
  if (out.x_host) {
    b->h_active.assign(count, 1);
    b->h_sent.assign(count, 0);
    if (stream_download(b, x, out, dl_call++, false, stream)) return 1;
  }
  if (*b->h_nactive > 0) {
    if (b->vcycle(L - 1, b->r, b->s, b->partial, act)) return 1;
    count_launch();
    pcg_rs_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->rs, b->active);
    const double* beta = nullptr;
    for (int k = 0; k < l_max; ++k) {
      count_launch();
      pcg_xpby_kernel<<<vg, 256, 0, stream>>>(n3, b->s, beta, b->p, b->active);
      e = coarse_launch(0, op, b->theta, count, b->p, nullptr, b->t_res, 0.0, act);
      if (e == cudaSuccess) e = vec_dot(n, count, b->p, n3, b->t_res, n3, b->partial, act);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      count_launch();
      pcg_alpha_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->rs,
                                                             b->alpha, b->active, b->pstatus);
      count_launch();
      pcg_update_kernel<<<vg, 256, 0, stream>>>(n3, b->p, b->t_res, b->alpha, x, b->r, b->active);
      e = vec_dot(n, count, b->r, n3, b->r, n3, b->partial, act);
      if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      count_launch();
      pcg_check_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->scale,
                                                             delta, l_max, b->hist, hl, b->active,
                                                             b->iters, b->nactive);
      if (dl_flush(b, x, out)) return 1;  // (behind this iteration's launches)
      e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      if (*b->h_nactive == 0) break;
      if (out.x_host && *b->h_nactive < b->cur_active &&
          dl_mark(b, out, dl_call++, false, stream))
        return 1;
      b->cur_active = *b->h_nactive;
      if (b->vcycle(L - 1, b->r, b->s, b->partial, act)) return 1;
      count_launch();
      pcg_beta_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->rs,
                                                            b->beta, b->active);
      beta = b->beta;
    }
  }
  if (out.x_host && stream_download(b, x, out, dl_call++, true, stream)) return 1;
  e = coarse_launch(1, op, b->theta, count, x, f, b->t_res, 0.0, all);
  if (e == cudaSuccess) e = vec_dot(n, count, b->t_res, n3, b->t_res, n3, b->partial, all);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  double* d_true = b->beta;
  count_launch();
  pcg_true_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->scale, d_true);
  e = cudaGetLastError();
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  std::vector<double> hh((size_t)count * hl);
  e = fetch_to_host(hh.data(), b->hist, sizeof(double) * count * hl, stream);
  if (e == cudaSuccess && out.iters) e = fetch_to_host(out.iters, b->iters, sizeof(int) * count, stream);
  if (e == cudaSuccess && out.true_res)
    e = fetch_to_host(out.true_res, d_true, sizeof(double) * count, stream);
  if (e == cudaSuccess && out.status)
    e = fetch_to_host(out.status, b->pstatus, sizeof(int) * count, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  const int hist_len = l_max + 1;
  if (out.hist)
    for (int m = 0; m < count; ++m)
      memcpy(out.hist + (size_t)m * hist_len, hh.data() + (size_t)m * hl, sizeof(double) * hist_len);
  if (out.status && out.true_res)
    for (int m = 0; m < count; ++m)
      if (!(out.status[m] & 1) && !(out.true_res[m] <= delta)) out.status[m] |= 2;
  return 0;
}

int pcg_solve(Batch* b, const double* f, int64_t f_stride, double* x, double delta, int l_max,
              const PcgOut& out, cudaStream_t stream) {
  if (!(delta > 0)) RBWS_FAIL("tolerance must be positive");
  if (l_max < 0) RBWS_FAIL("l_max must be non-negative");
  Hierarchy* h = b->h;
  const int count = b->count;
  if (count < 1) RBWS_FAIL("batch_setup must be called before solving");
  const int n = h->n;
  const int L = h->levels;
  const int hist_len = l_max + 1;
  cudaError_t e = cudaSuccess;
  if (hist_len * b->cap > b->hist_len * b->cap || !b->hist) {
    cudaFree(b->hist);
    e = dalloc(&b->hist, (size_t)b->cap * hist_len);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    b->hist_len = hist_len;
  }
  const int hl = b->hist_len;
  if (h->stored) return pcg_solve_stored(b, f, f_stride, x, delta, l_max, out, stream);
  const Sep7 op = b->fine_op();
  bool graph_ran = false;
  const int tiles = fine_geom(n, count).tiles;
  // the V-cycle's dot partials come from the post-smoothing kernel's geometry (nu = 1)
  const int vtiles = (b->smoother == 1) ? vec_tiles(n)
                     : ((b->nu == 1) ? fine_post_tiles(n, count) : tiles);
  LaunchCtx all{stream, nullptr};
  LaunchCtx act{stream, b->active};
  const int fshared = (f_stride == 0);
  const int ftiles = vec_tiles(n);
  // ||f||
  e = vec_dot(n, fshared ? 1 : count, f, f_stride, f, f_stride, b->partial2, all);
  // r = f - A x0, ||r||^2  (a shared rhs is staged once per plane for every instance)
  b->rcur = b->r;
  b->cgp_used = cgp_ok(b, op, act);
  if (b->cgp_used && !b->r2) {  // second residual buffer of the fused CG update
    e = dalloc(&b->r2, (size_t)vec_doubles(n, b->cap));
    if (e == cudaSuccess) e = cudaMemsetAsync(b->r2, 0, sizeof(double) * vec_doubles(n, b->cap), stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  }
  if (e == cudaSuccess) e = fine_resid(op, count, x, f, b->r, b->partial, all, fshared);
  if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  count_launch();
  pcg_init_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial2, ftiles, fshared,
                                                        b->partial, tiles, delta, l_max, b->scale,
                                                        b->hist, hl, b->active, b->iters,
                                                        b->pstatus, b->nactive);
  e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  b->cur_active = *b->h_nactive;
  int dl_call = 0;
  if (out.x_host) {
    b->h_active.assign(count, 1);
    b->h_sent.assign(count, 0);
    if (stream_download(b, x, out, dl_call++, false, stream)) return 1;  // converged at x0
  }
  if (*b->h_nactive > 0) {
    if (b->vcycle(L - 1, b->r, b->s, b->partial, act)) return 1;
    count_launch();
    pcg_rs_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, vtiles, b->rs, b->active);
    // search directions ping-pong between p and p2 (the p-update reads the old
    // direction with a halo, so it cannot be updated in place)
    double* p_old = nullptr;
    double* p_new = b->p;
    const double* beta = nullptr;
    const bool pf = b->prof_on;
    // the device-side loop has no per-iteration host readback: not with the event
    // profiler or the streaming download, which act on the host between iterations
    const bool use_graph = b->use_graph && !pf && !out.x_host;
    for (int k = 0; k < l_max; ++k) {
      int t0 = pf ? b->prof_begin(stream) : -1;
      e = fine_papply(op, count, b->s, p_old, beta, p_new, b->partial, act);
      if (pf) { b->prof_end(PROF_FINE_APPLY_DOT, t0, stream); t0 = b->prof_begin(stream); }
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      count_launch();
      pcg_alpha_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->rs,
                                                             b->alpha, b->active, b->pstatus);
      if (pf) { b->prof_end(PROF_SCALARS, t0, stream); t0 = b->prof_begin(stream); }
      const bool cgp = cgp_ok(b, op, act);
      if (cgp) {
        double* r_out = (b->rcur == b->r) ? b->r2 : b->r;
        e = fine_cg_update_pre(op, count, p_new, x, b->rcur, r_out, b->alpha, b->partial,
                               b->lv[L - 1].t1, b->omega, act);
        b->rcur = r_out;
      } else {
        e = fine_cg_update(op, count, p_new, x, b->rcur, b->alpha, b->partial, act);
      }
      if (pf) { b->prof_end(PROF_FINE_CG_UPDATE, t0, stream); t0 = b->prof_begin(stream); }
      if (e == cudaSuccess) e = cudaMemsetAsync(b->nactive, 0, sizeof(int), stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      count_launch();
      pcg_check_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->scale,
                                                             delta, l_max, b->hist, hl, b->active,
                                                             b->iters, b->nactive);
      if (pf) b->prof_end(PROF_SCALARS, t0, stream);
      if (dl_flush(b, x, out)) return 1;  // (behind this iteration's launches)
      e = fetch_to_host(b->h_nactive, b->nactive, sizeof(int), stream);
      if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
      if (*b->h_nactive == 0) break;
      // instances that stopped this iteration: their x is final; claim them now, enqueue
      // the copies once the next iteration's kernels are launched
      if (out.x_host && *b->h_nactive < b->cur_active &&
          dl_mark(b, out, dl_call++, false, stream))
        return 1;
      b->cur_active = *b->h_nactive;
      b->pre_done = cgp;
      const int vrc = b->vcycle(L - 1, b->rcur, b->s, b->partial, act);
      b->pre_done = false;
      if (vrc) return 1;
      if (pf) t0 = b->prof_begin(stream);
      count_launch();
      pcg_beta_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, vtiles, b->rs,
                                                            b->beta, b->active);
      if (pf) b->prof_end(PROF_SCALARS, t0, stream);
      beta = b->beta;
      p_old = p_new;
      p_new = (p_new == b->p) ? b->p2 : b->p;
      if (use_graph && k == 0 && k + 1 < l_max) {  // iterations 1.. on the device
        if (pcg_graph_run(b, op, x, tiles, vtiles, delta, l_max, hl, act, stream)) return 1;
        graph_ran = true;
        break;
      }
    }
  }
  // the rest (last to converge, l_max reached, breakdown)
  if (out.x_host && stream_download(b, x, out, dl_call++, true, stream)) return 1;
  // true residual ||f - A x|| / scale for every instance (the norm only: no vector written)
  if (e == cudaSuccess) e = fine_resid(op, count, x, f, nullptr, b->partial, all, fshared);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  double* d_true = b->beta;  // reuse as scratch
  count_launch();
  pcg_true_kernel<<<warp_grid(count), 256, 0, stream>>>(count, b->partial, tiles, b->scale, d_true);
  e = cudaGetLastError();
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  // results to host
  std::vector<double> hh((size_t)count * hl);
  // (zero-copy readbacks: they must not queue behind bulk DMA on the copy engines)
  e = fetch_to_host(hh.data(), b->hist, sizeof(double) * count * hl, stream);
  if (e == cudaSuccess && out.iters) e = fetch_to_host(out.iters, b->iters, sizeof(int) * count, stream);
  if (e == cudaSuccess && out.true_res)
    e = fetch_to_host(out.true_res, d_true, sizeof(double) * count, stream);
  if (e == cudaSuccess && out.status)
    e = fetch_to_host(out.status, b->pstatus, sizeof(int) * count, stream);
  if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
  if (graph_ran) {  // launches replayed by the graph: body x replays
    std::vector<int> it(count);
    e = fetch_to_host(it.data(), b->iters, sizeof(int) * count, stream);
    if (e != cudaSuccess) RBWS_FAIL(cudaGetErrorString(e));
    const int mx = *std::max_element(it.begin(), it.end());
    count_launches((int64_t)std::max(1, mx / 2) * b->gbody_launches);
  }
  if (b->prof_on) b->prof_flush();
  if (out.hist)
    for (int m = 0; m < count; ++m)
      memcpy(out.hist + (size_t)m * hist_len, hh.data() + (size_t)m * hl, sizeof(double) * hist_len);
  if (out.status && out.true_res)
    for (int m = 0; m < count; ++m)
      if (!(out.status[m] & 1) && !(out.true_res[m] <= delta)) out.status[m] |= 2;
  return 0;
}

}  // namespace rbws
