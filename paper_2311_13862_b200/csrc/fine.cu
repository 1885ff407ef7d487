// Finest-level kernels with TMA-engine plane staging (sm_100a).
//
// A CTA owns TY full grid rows of one parameter instance (one thread per grid
// column (i, j)) and marches through a z-range.  The TY rows of a plane, plus
// one halo row above and below for stencil inputs, form ONE contiguous byte
// range, staged into shared memory with a single cp.async.bulk per array per
// plane (TMA engine, completion on an mbarrier).  An 8-slot ring keeps planes
// k-1, k, k+1 resident while planes k+2..k+6 are in flight; every neighbour
// read is a shared-memory read and global memory sees each byte once (halo
// rows are L2 hits of the neighbouring tile).
//
// The separable affine operator is matrix-free: each thread holds 5Q column
// constants theta_q * (x/y factors) in registers; a face weight is
// sum_q const_q * zfactor_q(k).  The z factors of the CTA's planes live in
// shared memory with a per-plane flag telling whether they repeat the previous
// plane's; for piecewise-constant (thermal-block) coefficients they almost
// always do, so the six face weights and the diagonal stay cached in
// registers and a node costs only the 7-point update.
#include "fine.cuh"
#include "tma.cuh"

namespace rbws {

constexpr int kStages = 8;  // ring slots (power of two)
constexpr int kMaxKz = 64;  // planes per z-chunk (bounds the z-factor table)
constexpr int kThreads = 256;  // threads per CTA (one per grid column of the tile)

FineGeom fine_geom(int n, int batch) {
  FineGeom g;
  int rpp = kThreads / n;
  if (rpp < 1) rpp = 1;
  if (rpp > n) rpp = n;
  g.rpp = rpp;
  g.npt = (rpp * 2 <= n) ? 2 : 1;
  g.ty = rpp * g.npt;
  g.threads = rpp * n;
  g.ytiles = n / g.ty;
  g.zc = 1;
  while (n / g.zc > kMaxKz) g.zc *= 2;
  while ((int64_t)g.ytiles * batch * g.zc < 2 * 148 && (n / (g.zc * 2)) >= 8) g.zc *= 2;
  g.tiles = g.ytiles * g.zc;
  return g;
}

struct FineArgs {
  Sep7 op;
  FineGeom g;
  int dot;
  const double* h0;  // staged with halo rows
  const double* h1;
  const double* c0;  // staged, tile rows only
  const double* c1;
  double* out0;
  double* out1;
  const double* scal;  // per-instance scalar (alpha / beta)
  double* partial;
  const int* active;
  double omega;
  int c0_shared;  // c0 is one instance shared by the whole batch (e.g. the rhs f)
};

enum FineMode : int {
  FM_APPLY = 0,   // h0 = x                  out0 = A x (optional), dot x.Ax
  FM_RESID = 1,   // h0 = x, c0 = b          out0 = b - A x, dot |r|^2
  FM_JACOBI = 2,  // h0 = x, c0 = b          out0 = x + w (b - A x)/d, dot b.out
  FM_PRE = 3,     // h0 = b, h1 = dinv       out0 = b - A (w dinv b)
  FM_CG = 4,      // h0 = p, c0 = x, c1 = r  x += a p, r -= a A p (in place), dot |r|^2
  FM_PAPPLY = 5,  // h0 = s, h1 = p_old      out0 = p = s + b p_old, dot p.Ap
};

template <int MODE>
struct SL {
  static constexpr int NH = (MODE == FM_PRE || MODE == FM_PAPPLY) ? 2 : 1;
  static constexpr int NC = (MODE == FM_CG) ? 2 : ((MODE == FM_RESID || MODE == FM_JACOBI) ? 1 : 0);
};

template <int Q, int MODE, int NPT>
__global__ void __launch_bounds__(kThreads) fine_kernel(FineArgs a) {
  constexpr int NH = SL<MODE>::NH, NC = SL<MODE>::NC, S = kStages, ZW = 3 * Q;
  extern __shared__ __align__(128) unsigned char smem[];
  const Sep7& op = a.op;
  const int n = op.n, n1 = n + 1;
  const int ty = a.g.ty, zc = a.g.zc;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (a.active && !a.active[mu]) return;
  const int yt = blockIdx.y;
  const int j0 = yt * ty;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t n2 = (int64_t)n * n;
  const int64_t base = (int64_t)mu * n2 * n;
  const int kz = n / zc;
  const int kb = max(1, kc * kz), ke = min(n, (kc + 1) * kz);
  const int p_first = kb - 1, p_last = ke;  // staged planes (inclusive)
  const int np = p_last - p_first + 1;

  // ---- shared memory carve-up (offsets multiples of 16 bytes)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);            // [S]
  int* zsame = reinterpret_cast<int*>(smem + 64);                // [kMaxKz + 2]
  double* zf = reinterpret_cast<double*>(smem + 64 + 4 * (kMaxKz + 4));  // [np][3Q]
  double* ring = zf + ((np * ZW + 1) & ~1);
  const int hsz = (ty + 2) * n, csz = ty * n;
  const int stage_d = NH * hsz + NC * csz;
  auto hptr = [&](int st, int arr) { return ring + st * stage_d + arr * hsz; };
  auto cptr = [&](int st, int arr) { return ring + st * stage_d + NH * hsz + arr * csz; };

  for (int t = tid; t < np * ZW; t += nthr) {  // z factors of the staged planes
    const int p = t / ZW, f = (t / Q) % 3, q = t % Q, k = p_first + p;
    const double* F = op.face + (size_t)q * 3 * n;
    const double* N = op.node + (size_t)q * 9 * n1;
    double v;
    if (f == 0) v = N[(0 * 3 + 2) * n1 + k];       // x-part along z
    else if (f == 1) v = N[(1 * 3 + 2) * n1 + k];  // y-part along z
    else v = (k < n) ? F[2 * n + k] : 0.0;         // z-face k, k+1
    zf[t] = v;
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  for (int p = 1 + tid; p < np; p += nthr) {  // plane p repeats plane p-1's z factors?
    int same = 1;
    for (int t = 0; t < ZW; ++t) same &= (zf[p * ZW + t] == zf[(p - 1) * ZW + t]);
    zsame[p] = same;
  }

  const double* hsrc[2] = {a.h0, a.h1};
  const double* csrc[2] = {a.c0, a.c1};
  auto issue = [&](int p) {
    const int st = (p - p_first) & (S - 1);
    const int skip = (j0 == 0) ? 1 : 0;
    const uint32_t hbytes = (uint32_t)((ty + 2 - skip) * n * 8);
    const uint32_t cbytes = (uint32_t)(ty * n * 8);
    mbar_arrive_expect_tx(&bar[st], NH * hbytes + NC * cbytes);
    const int64_t plane = base + (int64_t)p * n2;
#pragma unroll
    for (int h = 0; h < NH; ++h)
      bulk_g2s(hptr(st, h) + skip * n, hsrc[h] + plane + (int64_t)(j0 - 1 + skip) * n, hbytes,
               &bar[st]);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      bulk_g2s(cptr(st, c),
               csrc[c] + (c == 0 && a.c0_shared ? plane - base : plane) + (int64_t)j0 * n, cbytes,
               &bar[st]);
  };
  if (tid == 0)
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);

  // ---- this thread's column i and rows j = j0 + rl0 + r*rpp
  const int i = tid % n;
  const int rl0 = tid / n;
  const int rpp = a.g.rpp;
  const double* th = op.theta + (size_t)mu * Q;
  const double sc = a.scal ? a.scal[mu] : 0.0;
  const double om = a.omega;
  double acc = 0.0;
  // cached face weights per owned row (recomputed only when the z factors change)
  double wxp[NPT], wxm[NPT], wyp[NPT], wym[NPT], wzp[NPT], wzm[NPT], dg[NPT], wdi[NPT];
  auto weights = [&](int r, const double* zk, bool first_plane) {
    const int j = j0 + rl0 + r * rpp;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    if (i >= 1 && j >= 1) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double* F = op.face + (size_t)q * 3 * n;
        const double* N = op.node + (size_t)q * 9 * n1;
        const double t = th[q];
        const double tx = t * __ldg(N + (0 * 3 + 1) * n1 + j) * zk[q];          // theta N_xy(j) zx(k)
        const double tyv = t * __ldg(N + (1 * 3 + 0) * n1 + i) * zk[Q + q];     // theta N_yx(i) zy(k)
        const double tz = t * __ldg(N + (2 * 3 + 0) * n1 + i) * __ldg(N + (2 * 3 + 1) * n1 + j);
        a0 = fma(__ldg(F + 0 * n + i), tx, a0);
        a1 = fma(__ldg(F + 0 * n + i - 1), tx, a1);
        a2 = fma(__ldg(F + 1 * n + j), tyv, a2);
        a3 = fma(__ldg(F + 1 * n + j - 1), tyv, a3);
        a4 = fma(tz, zk[2 * Q + q], a4);
      }
    }
    wzm[r] = first_plane ? a4 : wzp[r];
    wxp[r] = a0; wxm[r] = a1; wyp[r] = a2; wym[r] = a3; wzp[r] = a4;
  };
#pragma unroll
  for (int r = 0; r < NPT; ++r) weights(r, zf, true);  // plane kb-1: its z face is wzm of kb

  mbar_wait(&bar[0], 0u);
  mbar_wait(&bar[1], 0u);
  // KB planes per trip: one CTA barrier and KB TMA issues amortised over KB nodes per row
  constexpr int KB = 2;
  for (int k0 = kb; k0 < ke; k0 += KB) {
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      const int k = k0 + u;
      if (k >= ke) break;
      const int idx = k + 1 - p_first;
      mbar_wait(&bar[idx & (S - 1)], (uint32_t)((idx / S) & 1));
      const bool fresh = (k == kb) || !zsame[k - p_first];  // CTA-uniform
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        if (fresh) {
          weights(r, zf + (k - p_first) * ZW, false);
          dg[r] = ((wxp[r] + wxm[r]) + (wyp[r] + wym[r])) + (wzp[r] + wzm[r]);
          wdi[r] = om / dg[r];  // cached damping / diagonal (no per-node division)
        } else if (wzm[r] != wzp[r]) {
          wzm[r] = wzp[r];
          dg[r] = ((wxp[r] + wxm[r]) + (wyp[r] + wym[r])) + (wzp[r] + wzm[r]);
          wdi[r] = om / dg[r];
        }
      }
      const int sm = (idx - 2) & (S - 1), s0 = (idx - 1) & (S - 1), sp = idx & (S - 1);
      const int64_t kofs = base + (int64_t)k * n2 + i;
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        const int jl = rl0 + r * rpp;
        const int j = j0 + jl;
        const int hi = (jl + 1) * n + i;
        const int ci = jl * n + i;
        double uc, ue, uw, un, us, uu, ud;
        if (MODE == FM_PRE) {
          const double* B0 = hptr(s0, 0); const double* D0 = hptr(s0, 1);
          const double* BM = hptr(sm, 0); const double* DM = hptr(sm, 1);
          const double* BP = hptr(sp, 0); const double* DP = hptr(sp, 1);
          uc = om * D0[hi] * B0[hi];
          ue = om * D0[hi + 1] * B0[hi + 1];
          uw = om * D0[hi - 1] * B0[hi - 1];
          un = om * D0[hi + n] * B0[hi + n];
          us = om * D0[hi - n] * B0[hi - n];
          uu = om * DP[hi] * BP[hi];
          ud = om * DM[hi] * BM[hi];
        } else if (MODE == FM_PAPPLY) {
          const double* X0 = hptr(s0, 0); const double* XM = hptr(sm, 0); const double* XP = hptr(sp, 0);
          const double* P0 = hptr(s0, 1); const double* PM = hptr(sm, 1); const double* PP = hptr(sp, 1);
          uc = fma(sc, P0[hi], X0[hi]);
          ue = fma(sc, P0[hi + 1], X0[hi + 1]);
          uw = fma(sc, P0[hi - 1], X0[hi - 1]);
          un = fma(sc, P0[hi + n], X0[hi + n]);
          us = fma(sc, P0[hi - n], X0[hi - n]);
          uu = fma(sc, PP[hi], XP[hi]);
          ud = fma(sc, PM[hi], XM[hi]);
        } else {
          const double* X0 = hptr(s0, 0); const double* XM = hptr(sm, 0); const double* XP = hptr(sp, 0);
          uc = X0[hi]; ue = X0[hi + 1]; uw = X0[hi - 1]; un = X0[hi + n]; us = X0[hi - n];
          uu = XP[hi]; ud = XM[hi];
        }
        // shallow FMA tree (a dependent chain of 6 would be latency bound)
        const double offx = fma(wxm[r], uw, wxp[r] * ue);
        const double offy = fma(wym[r], us, wyp[r] * un);
        const double offz = fma(wzm[r], ud, wzp[r] * uu);
        const double off = (offx + offy) + offz;
        const double d = dg[r];
        const double Au = fma(d, uc, -off);
        const bool on = (i != 0) && (j != 0);  // Dirichlet ghost column / row
        const int64_t gidx = kofs + (int64_t)j * n;
        if (MODE == FM_APPLY) {
          if (on && a.out0) a.out0[gidx] = Au;
          acc = on ? fma(uc, Au, acc) : acc;
        } else if (MODE == FM_RESID) {
          const double rv = cptr(s0, 0)[ci] - Au;
          if (on) a.out0[gidx] = rv;
          acc = on ? fma(rv, rv, acc) : acc;
        } else if (MODE == FM_JACOBI) {
          const double bv = cptr(s0, 0)[ci];
          const double y = fma(wdi[r], bv - Au, uc);
          if (on) a.out0[gidx] = y;
          acc = on ? fma(bv, y, acc) : acc;
        } else if (MODE == FM_PRE) {
          if (on) a.out0[gidx] = hptr(s0, 0)[hi] - Au;
        } else if (MODE == FM_CG) {
          const double xv = fma(sc, uc, cptr(s0, 0)[ci]);
          const double rv = fma(-sc, Au, cptr(s0, 1)[ci]);
          if (on) {
            a.out0[gidx] = xv;
            a.out1[gidx] = rv;
          }
          acc = on ? fma(rv, rv, acc) : acc;
        } else {  // FM_PAPPLY
          if (on) a.out0[gidx] = uc;
          acc = on ? fma(uc, Au, acc) : acc;
        }
      }
    }
    __syncthreads();  // every thread is done with planes k0-1 .. k0+KB-2
    if (tid == 0) {
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int pn = k0 - 1 + u + S;
        if (pn <= p_last) issue(pn);
      }
    }
  }
  if (a.dot != DOT_NONE) {
    __shared__ double red[32];
    const double s = block_reduce_sum(acc, red);
    if (tid == 0) a.partial[(int64_t)mu * a.g.tiles + yt * zc + kc] = s;
  }
}

template <int Q, int MODE, int NPT>
static cudaError_t fine_launch_qmn(const FineArgs& a, int batch, cudaStream_t stream) {
  using L = SL<MODE>;
  const int n = a.op.n, ty = a.g.ty;
  const int np = n / a.g.zc + 2;
  const size_t stage_bytes = (size_t)(L::NH * (ty + 2) + L::NC * ty) * n * 8;
  const size_t smem = 64 + 4 * (kMaxKz + 4) + 8 * (((size_t)np * 3 * Q + 1) & ~(size_t)1) +
                      kStages * stage_bytes;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(fine_kernel<Q, MODE, NPT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  dim3 grd(1, a.g.ytiles, batch * a.g.zc);
  count_launch();
  fine_kernel<Q, MODE, NPT><<<grd, a.g.threads, smem, stream>>>(a);
  return cudaGetLastError();
}

template <int Q, int MODE>
static cudaError_t fine_launch_qm(const FineArgs& a, int batch, cudaStream_t stream) {
  if (a.g.npt == 2) return fine_launch_qmn<Q, MODE, 2>(a, batch, stream);
  if (a.g.npt == 1) return fine_launch_qmn<Q, MODE, 1>(a, batch, stream);
  return cudaErrorInvalidValue;
}

template <int Q>
static cudaError_t fine_launch_q(int mode, const FineArgs& a, int batch, cudaStream_t stream) {
  switch (mode) {
    case FM_APPLY: return fine_launch_qm<Q, FM_APPLY>(a, batch, stream);
    case FM_RESID: return fine_launch_qm<Q, FM_RESID>(a, batch, stream);
    case FM_JACOBI: return fine_launch_qm<Q, FM_JACOBI>(a, batch, stream);
    case FM_PRE: return fine_launch_qm<Q, FM_PRE>(a, batch, stream);
    case FM_CG: return fine_launch_qm<Q, FM_CG>(a, batch, stream);
    case FM_PAPPLY: return fine_launch_qm<Q, FM_PAPPLY>(a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

static cudaError_t fine_launch(int mode, FineArgs& a, int batch, cudaStream_t stream) {
  if (a.op.n > 256 || a.op.n < 8) return cudaErrorInvalidValue;
  a.g = fine_geom(a.op.n, batch);
  switch (a.op.Q) {
    case 1: return fine_launch_q<1>(mode, a, batch, stream);
    case 2: return fine_launch_q<2>(mode, a, batch, stream);
    case 3: return fine_launch_q<3>(mode, a, batch, stream);
    case 4: return fine_launch_q<4>(mode, a, batch, stream);
    case 5: return fine_launch_q<5>(mode, a, batch, stream);
    case 6: return fine_launch_q<6>(mode, a, batch, stream);
    case 7: return fine_launch_q<7>(mode, a, batch, stream);
    case 8: return fine_launch_q<8>(mode, a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

// 1/diag of the finest operator for every instance (batch setup); weights are
// recomputed only on planes whose z factors change (host-built flags)
template <int Q>
__global__ void __launch_bounds__(256) fine_dinv_kernel(Sep7 op, FineGeom g, const int* zsame,
                                                       double* __restrict__ dinv) {
  const int n = op.n, n1 = n + 1;
  const int kc = blockIdx.z % g.zc, mu = blockIdx.z / g.zc;
  const int kz = n / g.zc;
  const int kb = max(1, kc * kz), ke = min(n, (kc + 1) * kz);
  const int i = threadIdx.x % n;
  const int64_t n2 = (int64_t)n * n, base = (int64_t)mu * n2 * n;
  const double* th = op.theta + (size_t)mu * Q;
  for (int r = 0; r < g.npt; ++r) {
    const int j = blockIdx.y * g.ty + threadIdx.x / n + r * g.rpp;
    if (i == 0 || j == 0) continue;
    double d = 0.0;
    for (int k = kb; k < ke; ++k) {
      if (k == kb || !zsame[k]) {
        d = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double* F = op.face + (size_t)q * 3 * n;
          const double* N = op.node + (size_t)q * 9 * n1;
          const double xy = N[(0 * 3 + 1) * n1 + j] * N[(0 * 3 + 2) * n1 + k];
          const double yx = N[(1 * 3 + 0) * n1 + i] * N[(1 * 3 + 2) * n1 + k];
          const double zz = N[(2 * 3 + 0) * n1 + i] * N[(2 * 3 + 1) * n1 + j];
          const double s = (F[0 * n + i] + F[0 * n + i - 1]) * xy +
                           (F[1 * n + j] + F[1 * n + j - 1]) * yx +
                           (F[2 * n + k] + F[2 * n + k - 1]) * zz;
          d = fma(th[q], s, d);
        }
      }
      dinv[base + (int64_t)k * n2 + (int64_t)j * n + i] = 1.0 / d;
    }
  }
}

cudaError_t fine_dinv(const Sep7& op, int batch, const int* zsame, double* dinv,
                      cudaStream_t stream) {
  const FineGeom g = fine_geom(op.n, batch);
  dim3 grd(1, g.ytiles, batch * g.zc);
  count_launch();
#define RBWS_DQ(QQ) \
  case QQ: fine_dinv_kernel<QQ><<<grd, g.threads, 0, stream>>>(op, g, zsame, dinv); break;
  switch (op.Q) {
    RBWS_DQ(1) RBWS_DQ(2) RBWS_DQ(3) RBWS_DQ(4) RBWS_DQ(5) RBWS_DQ(6) RBWS_DQ(7) RBWS_DQ(8)
    default: return cudaErrorInvalidValue;
  }
#undef RBWS_DQ
  return cudaGetLastError();
}

static FineArgs base_args(const Sep7& op, int dot, double* partial, const LaunchCtx& lc,
                          double omega) {
  FineArgs a{};
  a.op = op;
  a.dot = dot;
  a.partial = partial;
  a.active = lc.active;
  a.omega = omega;
  return a;
}

cudaError_t fine_apply(const Sep7& op, int batch, const double* x, double* y, double* partial,
                       const LaunchCtx& lc) {
  FineArgs a = base_args(op, partial ? DOT_XAX : DOT_NONE, partial, lc, 0.0);
  a.h0 = x;
  a.out0 = y;
  return fine_launch(FM_APPLY, a, batch, lc.stream);
}

cudaError_t fine_resid(const Sep7& op, int batch, const double* x, const double* b, double* r,
                       double* partial, const LaunchCtx& lc, bool b_shared) {
  FineArgs a = base_args(op, partial ? DOT_YY : DOT_NONE, partial, lc, 0.0);
  a.h0 = x;
  a.c0 = b;
  a.c0_shared = b_shared ? 1 : 0;
  a.out0 = r;
  return fine_launch(FM_RESID, a, batch, lc.stream);
}

cudaError_t fine_jacobi(const Sep7& op, int batch, const double* x, const double* b, double* y,
                        double omega, double* partial, const LaunchCtx& lc) {
  FineArgs a = base_args(op, partial ? DOT_BY : DOT_NONE, partial, lc, omega);
  a.h0 = x;
  a.c0 = b;
  a.out0 = y;
  return fine_launch(FM_JACOBI, a, batch, lc.stream);
}

cudaError_t fine_pre(const Sep7& op, int batch, const double* b, const double* dinv, double* r1,
                     double omega, const LaunchCtx& lc) {
  FineArgs a = base_args(op, DOT_NONE, nullptr, lc, omega);
  a.h0 = b;
  a.h1 = dinv;
  a.out0 = r1;
  return fine_launch(FM_PRE, a, batch, lc.stream);
}

cudaError_t fine_cg_update(const Sep7& op, int batch, const double* p, double* x, double* r,
                           const double* alpha, double* partial, const LaunchCtx& lc) {
  FineArgs a = base_args(op, DOT_YY, partial, lc, 0.0);
  a.h0 = p;
  a.c0 = x;
  a.c1 = r;
  a.out0 = x;
  a.out1 = r;
  a.scal = alpha;
  return fine_launch(FM_CG, a, batch, lc.stream);
}

cudaError_t fine_papply(const Sep7& op, int batch, const double* s, const double* p_old,
                        const double* beta, double* p_new, double* partial, const LaunchCtx& lc) {
  FineArgs a = base_args(op, DOT_XAX, partial, lc, 0.0);
  a.h0 = s;
  a.h1 = p_old ? p_old : s;
  a.scal = beta;  // null (first iteration) -> p = s (h1 aliases s, weight 0)
  a.out0 = p_new;
  return fine_launch(FM_PAPPLY, a, batch, lc.stream);
}

}  // namespace rbws
