// Slab-decomposed MGCG for one large instance (BASELINE configs[4]: 512^3,
// slabs along z, one-plane halo exchange per stencil sweep).
//
// The reference solves one instance with pcg_solve + mg_vcycle (krylov.py:42-109,
// multigrid.py:205-232); this is the same algorithm with the grid of every fine
// level cut into R slabs of whole z-planes.  Slab r owns the planes
// [r n_l / R, (r+1) n_l / R) of level l and stores them with one halo plane on each
// side in the padded layout, so the finest-level and coarse-level kernels run
// unchanged on a slab: they receive "virtual" base pointers (plane k at V + k n^2)
// and the z-range of the owned planes (LaunchCtx::zlo/zhi).
//
// Communication, per V-cycle level and PCG iteration, is exactly what the stencils
// need: one halo plane in each direction of the vector a kernel reads with its
// 7/27-point stencil (refreshed after the kernel that wrote it), the lower halo of
// the pre-smoothing residual before the restriction, and an all-gather of the
// per-CTA dot-product partials (summed afterwards in a fixed order, so every slab
// computes bitwise identical scalars).  Levels with fewer than kMinSlabPlanes planes
// per slab are replicated: the restriction into the first replicated level writes
// each slab's own coarse planes and an all-gather completes the vector, below which
// every process runs the batched V-cycle (Batch::vcycle) on the whole level.
//
// Slabs of one process exchange halos with device copies; slabs of different
// processes (one per GPU) use NCCL send/recv over NVLink (comm.cu).
#include <algorithm>
#include <cstring>

#include "coarse.cuh"
#include "fine.cuh"
#include "slab.cuh"

#define RBWS_FAIL(msg) return rbws_set_error(msg, __FILE__, __LINE__)
#define RBWS_CK(expr)                                                        \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return rbws_set_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

namespace rbws {

constexpr int kMinSlabPlanes = 8;  // coarse levels with fewer planes per slab are replicated

Slab::~Slab() {
  for (auto& p : parts)
    for (auto& lv : p.v)
      for (double* b : lv) cudaFree(b);
  delete rep;
  delete comm;
  for (void* q : {(void*)theta, (void*)partial, (void*)partial2, (void*)rs, (void*)alpha,
                  (void*)beta, (void*)scale, (void*)tres, (void*)hist, (void*)active,
                  (void*)iters, (void*)status, (void*)nactive})
    cudaFree(q);
  cudaFreeHost(h_nactive);
}

double* Slab::V(const SlabPart& p, int l, int vid) const {
  const int64_t n2 = (int64_t)cells(l) * cells(l);
  return p.v[l][vid] - (int64_t)(p.k0[l] - 1) * n2;
}

LaunchCtx Slab::lc(const SlabPart& p, int l, cudaStream_t s, bool act) const {
  LaunchCtx c{s, act ? active : nullptr};
  c.zlo = p.k0[l];
  c.zhi = p.k1[l];
  return c;
}

// refresh halo planes of vector vid on level l: XCHG_UP sends every slab's top owned
// plane to the lower halo of the slab above, XCHG_DOWN the bottom owned plane to the
// upper halo of the slab below
int Slab::xchg(int l, int vid, int dirs, cudaStream_t s) {
  const int n = cells(l);
  const int64_t n2 = (int64_t)n * n;
  const int nz = n / R;
  const size_t bytes = (size_t)n2 * sizeof(double);
  const bool loop = comm && comm->nprocs == 1;  // NCCL loopback transport (tests)
  if (loop && comm_group_start()) return 1;
  for (int i = 0; i + 1 < nloc; ++i) {
    double* a = parts[i].v[l][vid];
    double* b = parts[i + 1].v[l][vid];
    if (loop) {  // the same NCCL send/recv pairs as between processes, to this rank
      if ((dirs & XCHG_UP) && (comm_send(comm, a + nz * n2, n2, 0, s) || comm_recv(comm, b, n2, 0, s)))
        return 1;
      if ((dirs & XCHG_DOWN) &&
          (comm_send(comm, b + n2, n2, 0, s) || comm_recv(comm, a + (nz + 1) * n2, n2, 0, s)))
        return 1;
      continue;
    }
    if (dirs & XCHG_UP)
      RBWS_CK(cudaMemcpyAsync(b, a + nz * n2, bytes, cudaMemcpyDeviceToDevice, s));
    if (dirs & XCHG_DOWN)
      RBWS_CK(cudaMemcpyAsync(a + (nz + 1) * n2, b + n2, bytes, cudaMemcpyDeviceToDevice, s));
  }
  if (loop && comm_group_end()) return 1;
  if (comm && comm->nprocs > 1) {
    const int pr = comm->rank, np = comm->nprocs;
    if (comm_group_start()) return 1;
    if (pr + 1 < np) {
      double* t = parts.back().v[l][vid];
      if ((dirs & XCHG_UP) && comm_send(comm, t + nz * n2, n2, pr + 1, s)) return 1;
      if ((dirs & XCHG_DOWN) && comm_recv(comm, t + (nz + 1) * n2, n2, pr + 1, s)) return 1;
    }
    if (pr > 0) {
      double* b = parts.front().v[l][vid];
      if ((dirs & XCHG_UP) && comm_recv(comm, b, n2, pr - 1, s)) return 1;
      if ((dirs & XCHG_DOWN) && comm_send(comm, b + n2, n2, pr - 1, s)) return 1;
    }
    if (comm_group_end()) return 1;
  }
  return 0;
}

int Slab::gather_partials(double* part, int tps, cudaStream_t s) {
  if (comm) return comm_allgather(comm, part, (size_t)nloc * tps, s);  // 1 process: identity
  return 0;
}

int Slab::vcycle(int l, int vb, int vout, bool dot, cudaStream_t st) {
  const bool fine = (l == L - 1);
  const int c = l - 1;
  const bool cdist = c >= Ld;
  const int n = cells(l), nc = cells(c);
  const Sep7 fop{h->n, h->Q, h->d_face, h->d_node, theta, h->fine_zchg, h->d_fzsame};
  // pre-smoothing from zero and its residual: t = b - A (w D^-1 b)
  if (fine) {
    for (auto& P : parts)
      RBWS_CK(fine_pre(fop, 1, V(P, l, vb), V(P, l, SV_DINV), V(P, l, SV_T), omega,
                       lc(P, l, st, true)));
  } else {
    if (xchg(l, SV_U, XCHG_BOTH, st)) return 1;
    for (auto& P : parts)
      RBWS_CK(coarse_launch(1, h->coarse_op(l), theta, 1, V(P, l, SV_U), V(P, l, vb),
                            V(P, l, SV_T), omega, lc(P, l, st, true)));
  }
  if (xchg(l, SV_T, XCHG_UP, st)) return 1;  // the restriction reads plane k0 - 1
  std::vector<const double*> ec(parts.size());
  if (cdist) {
    for (auto& P : parts)
      RBWS_CK(restrict_launch(n, 1, V(P, l, SV_T), V(P, c, SV_B), lc(P, c, st, true),
                              c >= 1 ? V(P, c, SV_DINV) : nullptr,
                              c >= 1 ? V(P, c, SV_U) : nullptr, omega));
    if (vcycle(c, SV_B, SV_E, false, st)) return 1;
    if (xchg(c, SV_E, XCHG_BOTH, st)) return 1;
    for (size_t i = 0; i < parts.size(); ++i) ec[i] = V(parts[i], c, SV_E);
  } else {
    LevelBuf& cb = rep->lv[c];
    for (auto& P : parts) {
      LaunchCtx cl{st, active};
      cl.zlo = P.k0[l] / 2;
      cl.zhi = P.k1[l] / 2;
      RBWS_CK(restrict_launch(n, 1, V(P, l, SV_T), cb.b, cl));
    }
    if (gather_partials(cb.b, (nc / R) * nc * nc, st)) return 1;  // planes, not partials
    if (c >= 1) RBWS_CK(vec_scale_dinv(nc, 1, omega, cb.dinv, cb.b, cb.u, st));
    LaunchCtx rl{st, active};
    if (rep->vcycle(c, cb.b, cb.e, nullptr, rl)) return 1;
    for (size_t i = 0; i < parts.size(); ++i) ec[i] = cb.e;
  }
  if (fine) {  // prolongation fused into the post-smoothing sweep
    for (size_t i = 0; i < parts.size(); ++i) {
      const SlabPart& P = parts[i];
      RBWS_CK(fine_post_prolong(fop, 1, V(P, l, vb), V(P, l, SV_DINV), ec[i], V(P, l, vout),
                                omega, dot ? partial + (int64_t)P.rank * vtiles : nullptr,
                                lc(P, l, st, true)));
    }
  } else {
    for (size_t i = 0; i < parts.size(); ++i) {
      const SlabPart& P = parts[i];
      RBWS_CK(prolong_launch(n, 1, 2, ec[i], V(P, l, SV_T), V(P, l, SV_U), nullptr, omega,
                             lc(P, l, st, true)));
    }
    if (xchg(l, SV_T, XCHG_BOTH, st)) return 1;
    for (auto& P : parts)
      RBWS_CK(coarse_launch(2, h->coarse_op(l), theta, 1, V(P, l, SV_T), V(P, l, vb),
                            V(P, l, vout), omega, lc(P, l, st, true)));
  }
  return 0;
}

template <class T>
static cudaError_t zalloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T) + 16);
  if (e == cudaSuccess) e = cudaMemset(*p, 0, count * sizeof(T) + 16);
  return e;
}

int slab_create(Slab** out, Hierarchy* h, int nslabs, int first, int nloc, Comm* comm,
                double omega) {
  const int L = h->levels, n = h->n;
  if (nslabs < 1 || nloc < 1 || first < 0 || first + nloc > nslabs)
    RBWS_FAIL("bad slab partition");
  const int nprocs = comm ? comm->nprocs : 1;
  if (nloc * nprocs != nslabs) RBWS_FAIL("every process must hold the same number of slabs");
  if (comm && first != comm->rank * nloc) RBWS_FAIL("slabs must be assigned in process order");
  if (n % (2 * nslabs) || n / nslabs < 4)
    RBWS_FAIL("finest grid needs an even number >= 4 of planes per slab");
  if (L < 2) RBWS_FAIL("slab solver needs at least two levels");
  Slab* s = new Slab();
  s->h = h; s->R = nslabs; s->nloc = nloc; s->first = first; s->L = L; s->omega = omega;
  s->comm = comm;
  int Ld = L - 1;
  while (Ld - 1 >= 1 && h->cells[Ld - 1] % nslabs == 0 &&
         h->cells[Ld - 1] / nslabs >= kMinSlabPlanes)
    --Ld;
  s->Ld = Ld;
  cudaError_t e = cudaSuccess;
  s->parts.resize(nloc);
  for (int i = 0; i < nloc && e == cudaSuccess; ++i) {
    SlabPart& P = s->parts[i];
    P.rank = first + i;
    P.k0.assign(L, 0);
    P.k1.assign(L, 0);
    P.v.resize(L);
    for (int l = 0; l < L; ++l) P.v[l].fill(nullptr);
    for (int l = Ld; l < L && e == cudaSuccess; ++l) {
      const int nl = h->cells[l], nz = nl / nslabs;
      P.k0[l] = P.rank * nz;
      P.k1[l] = (P.rank + 1) * nz;
      const size_t cnt = (size_t)(nz + 4) * nl * nl;  // halo planes + two-plane zero tail
      std::vector<int> ids;
      if (l == L - 1) ids = {SV_X, SV_F, SV_R, SV_P, SV_P2, SV_S, SV_T, SV_DINV};
      else ids = {SV_B, SV_E, SV_T, SV_DINV, SV_U};
      for (int id : ids)
        if (e == cudaSuccess) e = zalloc(&P.v[l][id], cnt);
    }
  }
  const int nz = n / nslabs;
  s->tiles = fine_geom(n, 1, nz).tiles;
  s->vtiles = fine_post_tiles(n, 1, nz);
  s->ftiles = (int)(((int64_t)nz * n * n + 2047) / 2048);
  if (e == cudaSuccess) e = zalloc(&s->theta, kMaxTerms);
  if (e == cudaSuccess)
    e = zalloc(&s->partial, (size_t)nslabs * std::max(s->tiles, s->vtiles));
  if (e == cudaSuccess) e = zalloc(&s->partial2, (size_t)nslabs * s->ftiles);
  for (double** pp : {&s->rs, &s->alpha, &s->beta, &s->scale, &s->tres})
    if (e == cudaSuccess) e = zalloc(pp, 1);
  for (int** pp : {&s->active, &s->iters, &s->status, &s->nactive})
    if (e == cudaSuccess) e = zalloc(pp, 1);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&s->h_nactive, sizeof(int));
  if (e != cudaSuccess) {
    s->comm = nullptr;  // owned by the caller until creation succeeds
    delete s;
    RBWS_FAIL(cudaGetErrorString(e));
  }
  if (batch_create(&s->rep, h, 1, 1, omega, Ld)) {
    s->comm = nullptr;
    delete s;
    return 1;
  }
  *out = s;
  return 0;
}

int slab_setup(Slab* s, const double* theta, int* n_bad, cudaStream_t st) {
  Hierarchy* h = s->h;
  const int L = s->L;
  RBWS_CK(cudaMemcpyAsync(s->theta, theta, sizeof(double) * h->Q, cudaMemcpyDefault, st));
  const Sep7 fop{h->n, h->Q, h->d_face, h->d_node, s->theta, h->fine_zchg, h->d_fzsame};
  for (auto& P : s->parts) {
    // finest 1/diag including the halo planes (the pre/post-smoothing kernels stage them)
    const int zlo = std::max(1, P.k0[L - 1] - 1), zhi = std::min(h->n, P.k1[L - 1] + 1);
    RBWS_CK(fine_dinv(fop, 1, h->d_fzsame, s->V(P, L - 1, SV_DINV), st, zlo, zhi));
    for (int l = s->Ld; l < L - 1; ++l)
      RBWS_CK(coarse_launch(4, h->coarse_op(l), s->theta, 1, nullptr, nullptr,
                            s->V(P, l, SV_DINV), 0.0, s->lc(P, l, st, false)));
  }
  if (batch_setup(s->rep, s->theta, 1, st)) return 1;
  int bad = 0;
  RBWS_CK(fetch_to_host(&bad, s->rep->d_status, sizeof(int), st));
  if (n_bad) *n_bad = bad ? 1 : 0;
  s->ready = true;
  return 0;
}

int slab_load(Slab* s, int vid, const double* src, int64_t p0, int planes, cudaStream_t st) {
  if (vid != SV_X && vid != SV_F) RBWS_FAIL("only x and f can be loaded");
  const int l = s->L - 1, n = s->h->n;
  const int64_t n2 = (int64_t)n * n;
  for (auto& P : s->parts) {
    const int64_t lo = std::max<int64_t>(P.k0[l], p0), hi = std::min<int64_t>(P.k1[l], p0 + planes);
    if (lo < hi)
      RBWS_CK(cudaMemcpyAsync(s->V(P, l, vid) + lo * n2, src + (lo - p0) * n2,
                              (size_t)((hi - lo) * n2) * sizeof(double), cudaMemcpyDefault, st));
  }
  return 0;
}

int slab_store(Slab* s, int vid, double* dst, int64_t p0, int planes, cudaStream_t st) {
  if (vid != SV_X && vid != SV_F) RBWS_FAIL("only x and f can be stored");
  const int l = s->L - 1, n = s->h->n;
  const int64_t n2 = (int64_t)n * n;
  for (auto& P : s->parts) {
    const int64_t lo = std::max<int64_t>(P.k0[l], p0), hi = std::min<int64_t>(P.k1[l], p0 + planes);
    if (lo < hi)
      RBWS_CK(cudaMemcpyAsync(dst + (lo - p0) * n2, s->V(P, l, vid) + lo * n2,
                              (size_t)((hi - lo) * n2) * sizeof(double), cudaMemcpyDefault, st));
  }
  return 0;
}

int slab_prolong_x(Slab* s, const double* ec, cudaStream_t st) {
  const int l = s->L - 1, n = s->h->n;
  const int64_t n2 = (int64_t)n * n;
  for (auto& P : s->parts) {
    double* x = s->V(P, l, SV_X);
    RBWS_CK(cudaMemsetAsync(x + P.k0[l] * n2, 0,
                            (size_t)(P.k1[l] - P.k0[l]) * n2 * sizeof(double), st));
    RBWS_CK(prolong_launch(n, 1, 0, ec, x, nullptr, nullptr, 0.0, s->lc(P, l, st, false)));
  }
  return 0;
}

int slab_solve(Slab* S, double delta, int l_max, int* iters, double* hist, double* true_res,
               int* status, cudaStream_t st) {
  if (!S->ready) RBWS_FAIL("slab_setup must be called before solving");
  if (!(delta > 0)) RBWS_FAIL("tolerance must be positive");
  if (l_max < 0) RBWS_FAIL("l_max must be non-negative");
  Hierarchy* h = S->h;
  const int L = S->L, l = L - 1, n = h->n, R = S->R;
  const int64_t n2 = (int64_t)n * n;
  const int nz = n / R;
  if (l_max + 1 > S->hist_len) {
    cudaFree(S->hist);
    S->hist = nullptr;
    RBWS_CK(zalloc(&S->hist, (size_t)l_max + 1));
    S->hist_len = l_max + 1;
  }
  const int hl = S->hist_len;
  const Sep7 op{n, h->Q, h->d_face, h->d_node, S->theta, h->fine_zchg, h->d_fzsame};
  const int T = S->tiles, VT = S->vtiles;  // VT: the V-cycle's (post-smoothing) dot slots
  auto part_of = [&](const SlabPart& P) { return S->partial + (int64_t)P.rank * T; };
  // ||f||^2 over the owned planes, r = f - A x0, |r|^2
  for (auto& P : S->parts)
    RBWS_CK(vec_dot_range((int64_t)nz * n2, S->V(P, l, SV_F) + P.k0[l] * n2,
                          S->V(P, l, SV_F) + P.k0[l] * n2,
                          S->partial2 + (int64_t)P.rank * S->ftiles, st));
  if (S->gather_partials(S->partial2, S->ftiles, st)) return 1;
  if (S->xchg(l, SV_X, XCHG_BOTH, st)) return 1;
  for (auto& P : S->parts)
    RBWS_CK(fine_resid(op, 1, S->V(P, l, SV_X), S->V(P, l, SV_F), S->V(P, l, SV_R), part_of(P),
                       S->lc(P, l, st, false)));
  if (S->gather_partials(S->partial, T, st)) return 1;
  RBWS_CK(cudaMemsetAsync(S->nactive, 0, sizeof(int), st));
  RBWS_CK(pcg_init(1, S->partial2, R * S->ftiles, 0, S->partial, R * T, delta, l_max, S->scale,
                   S->hist, hl, S->active, S->iters, S->status, S->nactive, st));
  RBWS_CK(fetch_to_host(S->h_nactive, S->nactive, sizeof(int), st));
  if (*S->h_nactive > 0) {
    if (S->xchg(l, SV_R, XCHG_BOTH, st)) return 1;
    if (S->vcycle(l, SV_R, SV_S, true, st)) return 1;
    if (S->gather_partials(S->partial, VT, st)) return 1;
    RBWS_CK(pcg_rs(1, S->partial, R * VT, S->rs, S->active, st));
    int p_old = -1, p_new = SV_P;
    for (int k = 0; k < l_max; ++k) {
      if (S->xchg(l, SV_S, XCHG_BOTH, st)) return 1;
      for (auto& P : S->parts)
        RBWS_CK(fine_papply(op, 1, S->V(P, l, SV_S), p_old < 0 ? nullptr : S->V(P, l, p_old),
                            p_old < 0 ? nullptr : S->beta, S->V(P, l, p_new), part_of(P),
                            S->lc(P, l, st, true)));
      if (S->gather_partials(S->partial, T, st)) return 1;
      RBWS_CK(pcg_alpha(1, S->partial, R * T, S->rs, S->alpha, S->active, S->status, st));
      if (S->xchg(l, p_new, XCHG_BOTH, st)) return 1;
      for (auto& P : S->parts)
        RBWS_CK(fine_cg_update(op, 1, S->V(P, l, p_new), S->V(P, l, SV_X), S->V(P, l, SV_R),
                               S->alpha, part_of(P), S->lc(P, l, st, true)));
      if (S->gather_partials(S->partial, T, st)) return 1;
      RBWS_CK(cudaMemsetAsync(S->nactive, 0, sizeof(int), st));
      RBWS_CK(pcg_check(1, S->partial, R * T, S->scale, delta, l_max, S->hist, hl, S->active,
                        S->iters, S->nactive, st));
      RBWS_CK(fetch_to_host(S->h_nactive, S->nactive, sizeof(int), st));
      if (*S->h_nactive == 0) break;
      if (S->xchg(l, SV_R, XCHG_BOTH, st)) return 1;
      if (S->vcycle(l, SV_R, SV_S, true, st)) return 1;
      if (S->gather_partials(S->partial, VT, st)) return 1;
      RBWS_CK(pcg_beta(1, S->partial, R * VT, S->rs, S->beta, S->active, st));
      p_old = p_new;
      p_new = (p_new == SV_P) ? SV_P2 : SV_P;
    }
  }
  // true residual ||f - A x|| / scale
  if (S->xchg(l, SV_X, XCHG_BOTH, st)) return 1;
  for (auto& P : S->parts)
    RBWS_CK(fine_resid(op, 1, S->V(P, l, SV_X), S->V(P, l, SV_F), S->V(P, l, SV_T), part_of(P),
                       S->lc(P, l, st, false)));
  if (S->gather_partials(S->partial, T, st)) return 1;
  RBWS_CK(pcg_true(1, S->partial, R * T, S->scale, S->tres, st));
  std::vector<double> hh(hl);
  RBWS_CK(fetch_to_host(hh.data(), S->hist, sizeof(double) * hl, st));
  int it = 0, stt = 0;
  double tr = 0.0;
  RBWS_CK(fetch_to_host(&it, S->iters, sizeof(int), st));
  RBWS_CK(fetch_to_host(&tr, S->tres, sizeof(double), st));
  RBWS_CK(fetch_to_host(&stt, S->status, sizeof(int), st));
  if (!(stt & 1) && !(tr <= delta)) stt |= 2;
  if (iters) *iters = it;
  if (true_res) *true_res = tr;
  if (status) *status = stt;
  if (hist) memcpy(hist, hh.data(), sizeof(double) * (l_max + 1));
  return 0;
}

}  // namespace rbws
