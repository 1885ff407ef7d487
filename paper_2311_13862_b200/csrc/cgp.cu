// CG update fused with the next V-cycle's pre-smoothing residual and the x/z passes of its
// restriction (sm_100a):
//   x += alpha p,  r -= alpha A p,  |r|^2          (krylov.py:89-92)
//   r1 = r - A (w D^-1 r)                            (multigrid.py:218-219, the V-cycle's input is r)
//   t  = x/z restriction of r1                       (multigrid.py:220; y pass: restrict_y_kernel)
// in one z-marching pass: r is never re-read (42 instead of 50 B/node) and the pre-smoothing's
// instructions fill the issue slots the HBM-bound CG update leaves idle.
//
// A CTA owns TY = 16 full rows of one instance (512 threads, two rows per thread) and the whole
// z-range.  The new residual is needed on one halo row on each side of the tile, so A p is
// also evaluated there (the first / last row group carries a third node per plane) from p
// staged with two halo rows.  u = w D^-1 r_new of the tile + halo rows goes to a two-plane
// shared-memory ring; the pre-smoothing residual of plane k-1 is finished one plane behind the
// CG update: its in-plane part and the z-face below are taken before the weights move to
// plane k, the z-face above (weight = plane k's lower face) after u(k) is known.
#include <atomic>
#include <cstdlib>

#include "fine.cuh"
#include "tma.cuh"

namespace rbws {

namespace {

#ifndef RBWS_CGP_THREADS
#define RBWS_CGP_THREADS 512
#endif
constexpr int kCgpThreads = RBWS_CGP_THREADS;
#ifndef RBWS_CGP_S
#define RBWS_CGP_S 4
#endif
constexpr int kCgpS = RBWS_CGP_S;  // ring slots (planes of p, r and x in flight)
#ifndef RBWS_CGP_UNROLL
#define RBWS_CGP_UNROLL 1
#endif
constexpr int kCgpUnroll = RBWS_CGP_UNROLL;  // planes per unrolled trip of the main loop

struct CgpArgs {
  Sep7 op;
  const double* p;
  double* x;
  const double* rin;   // r before the update (read with one halo row each side of the tile)
  double* rout;        // r after the update: another buffer — a neighbouring tile may still
                       // have to read this tile's old rows as its halo
  double* t;           // [n/2][n][n/2] per instance
  const double* alpha;
  double* partial;
  int tiles;           // partial slots per instance (the CG update kernel's geometry)
  const int* active;
  double omega;
};

template <int N>
struct CgpGeom {
  static constexpr int RPP = kCgpThreads / N;  // row groups
  static constexpr int TY = 2 * RPP;           // rows per tile
  static constexpr int PSZ = (TY + 4) * N;     // p: rows j0-2 .. j0+TY+1
  static constexpr int RSZ = (TY + 2) * N;     // r: rows j0-1 .. j0+TY
  static constexpr int XSZ = TY * N;           // x: tile rows
  static constexpr int STAGE = PSZ + RSZ + XSZ;
  static constexpr int USZ = (TY + 2) * N;     // u ring plane (rows j0-1 .. j0+TY)
  static constexpr int CSZ = TY * N;
  static size_t bytes(int Q) {
    return 64 + 8 * (size_t)(((N + 1) * 3 * Q + 1) & ~1) +
           8 * ((size_t)kCgpS * STAGE + 2 * USZ + 2 * CSZ + 2) + 16 + 4 * (size_t)(N + 4);
  }
};

template <int N>
__global__ void __launch_bounds__(kCgpThreads, kCgpThreads <= 256 ? 2 : 1) cgp_kernel(CgpArgs a) {
  using G = CgpGeom<N>;
  constexpr int RPP = G::RPP, TY = G::TY, S = kCgpS;
  constexpr int PSZ = G::PSZ, RSZ = G::RSZ, STAGE = G::STAGE, USZ = G::USZ, CSZ = G::CSZ;
  constexpr int XSZ = G::XSZ;
  constexpr int64_t N2 = (int64_t)N * N;
  extern __shared__ __align__(128) unsigned char smem[];
  const Sep7& op = a.op;
  const int Q = op.Q, ZW = 3 * Q;
  const int mu = blockIdx.z, yt = blockIdx.y;
  if (a.active && !a.active[mu]) return;
  const int j0 = yt * TY, tid = threadIdx.x;
  const int64_t base = (int64_t)mu * N2 * N;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  static_assert(kCgpS <= 8, "the ring barriers occupy the first 64 bytes");
  double* zf = reinterpret_cast<double*>(smem + 64);   // [N + 1][3Q]
  double* ring = zf + (((N + 1) * ZW + 1) & ~1);        // [S][STAGE]
  double* uring = ring + S * STAGE;                     // [2][USZ]
  double* rbuf = uring + 2 * USZ;                       // [2][CSZ]
  uint32_t* zbits = reinterpret_cast<uint32_t*>(rbuf + 2 * CSZ + 2);  // [2] plane k repeats k-1
  int* zs = reinterpret_cast<int*>(zbits + 4);                          // [N + 1] (N > 64)

  for (int t = tid; t < (N + 1) * ZW; t += kCgpThreads) {  // z factors of planes 0 .. N
    const int k = t / (3 * Q), f = (t / Q) % 3, q = t % Q;
    const double* F = op.face + (size_t)q * 3 * N;
    const double* NF = op.node + (size_t)q * 9 * (N + 1);
    double v;
    if (f == 0) v = NF[(0 * 3 + 2) * (N + 1) + k];
    else if (f == 1) v = NF[(1 * 3 + 2) * (N + 1) + k];
    else v = (k < N) ? F[2 * N + k] : 0.0;
    zf[t] = v;
  }
  for (int t = tid; t < 2 * USZ; t += kCgpThreads) uring[t] = 0.0;  // u(0) = 0, never-written rows
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid < 64) {  // bit k: plane k repeats plane k-1's z factors (k >= 2)
    bool sm = tid >= 2 && tid < N;
    for (int t = 0; t < ZW && sm; ++t) sm = (zf[tid * ZW + t] == zf[(tid - 1) * ZW + t]);
    const uint32_t bits = __ballot_sync(0xffffffffu, sm);
    if ((tid & 31) == 0) zbits[tid >> 5] = bits;
  }
  if (N > 64)
    for (int k = tid; k <= N; k += kCgpThreads) {
      bool sm = k >= 2 && k < N;
      for (int t = 0; t < ZW && sm; ++t) sm = (zf[k * ZW + t] == zf[(k - 1) * ZW + t]);
      zs[k] = sm ? 1 : 0;
    }
  __syncthreads();
  const uint64_t zmask = ((uint64_t)zbits[1] << 32) | zbits[0];
  // staged rows below 0 do not exist for the first tile
  const int skp = (j0 == 0) ? 2 : 0, skr = (j0 == 0) ? 1 : 0;
  auto issue = [&](int p) {
    double* st = ring + (p % S) * STAGE;
    const uint32_t pb = (uint32_t)((TY + 4 - skp) * N * 8), rb = (uint32_t)((TY + 2 - skr) * N * 8);
    constexpr uint32_t xb = (uint32_t)(XSZ * 8);
    mbar_arrive_expect_tx(&bar[p % S], pb + rb + xb);
    const int64_t plane = base + (int64_t)p * N2;
    bulk_g2s(st + skp * N, a.p + plane + (int64_t)(j0 - 2 + skp) * N, pb, &bar[p % S]);
    bulk_g2s(st + PSZ + skr * N, a.rin + plane + (int64_t)(j0 - 1 + skr) * N, rb, &bar[p % S]);
    bulk_g2s(st + PSZ + RSZ, a.x + plane + (int64_t)j0 * N, xb, &bar[p % S]);
  };
  auto wait = [&](int p) { mbar_wait(&bar[p % S], (uint32_t)((p / S) & 1)); };
  if (tid == 0)
    for (int p = 0; p < S && p <= N; ++p) issue(p);

  // ---- node slots of this thread: two own rows and (first / last row group) one halo row
  const int i = tid % N, rl0 = tid / N;
  constexpr int NS = 3;
  int row[NS];  // tile-relative row: -1 .. TY
  row[0] = rl0;
  row[1] = rl0 + RPP;
  row[2] = (rl0 == 0) ? -1 : TY;
  const bool has3 = (rl0 == 0) || (rl0 == RPP - 1);
  bool on[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int j = j0 + row[s];
    on[s] = (s < 2 || has3) && i >= 1 && j >= 1 && j <= N - 1;
  }
  const double* th = op.theta + (size_t)mu * Q;
  const double al = a.alpha[mu], om = a.omega;
  double wxp[NS] = {}, wxm[NS] = {}, wyp[NS] = {}, wym[NS] = {}, wzp[NS] = {}, wzm[NS] = {};
  double dg[NS] = {}, wdi[NS] = {};
  auto weights = [&](int s, const double* zk) {  // fine_kernel::weights
    const int j = j0 + row[s];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    if (on[s]) {
#pragma unroll 2
      for (int q = 0; q < Q; ++q) {
        const double* F = op.face + (size_t)q * 3 * N;
        const double* NF = op.node + (size_t)q * 9 * (N + 1);
        const double t = th[q];
        const double tx = t * __ldg(NF + (0 * 3 + 1) * (N + 1) + j) * zk[q];
        const double tyv = t * __ldg(NF + (1 * 3 + 0) * (N + 1) + i) * zk[Q + q];
        const double tz = t * __ldg(NF + (2 * 3 + 0) * (N + 1) + i) * __ldg(NF + (2 * 3 + 1) * (N + 1) + j);
        a0 = fma(__ldg(F + 0 * N + i), tx, a0);
        a1 = fma(__ldg(F + 0 * N + i - 1), tx, a1);
        a2 = fma(__ldg(F + 1 * N + j), tyv, a2);
        a3 = fma(__ldg(F + 1 * N + j - 1), tyv, a3);
        a4 = fma(tz, zk[2 * Q + q], a4);
      }
    }
    wxp[s] = a0; wxm[s] = a1; wyp[s] = a2; wym[s] = a3; wzp[s] = a4;
  };
  auto diag = [&](int s) {
    dg[s] = ((wxp[s] + wxm[s]) + (wyp[s] + wym[s])) + (wzp[s] + wzm[s]);
    wdi[s] = on[s] ? om / dg[s] : 0.0;
  };
#pragma unroll
  for (int s = 0; s < NS; ++s) {  // plane 0: its z face (0, 1) is wzm of plane 1
    weights(s, zf);
    wzm[s] = wzp[s];
  }
  bool pend = false;
  auto same = [&](int k) -> bool {  // CTA-uniform
    return N <= 64 ? ((zmask >> k) & 1) != 0 : zs[k] != 0;
  };
  auto refresh = [&](int k) {  // fine_kernel::refresh
    if (k == 1 || !same(k)) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double prev = wzp[s];
        weights(s, zf + k * ZW);
        wzm[s] = prev;
        diag(s);
      }
      pend = true;
    } else if (pend) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        wzm[s] = wzp[s];
        diag(s);
      }
      pend = false;
    }
  };

  // offsets of the slots inside the staged p rows (first row = j0-2), r rows / u rows (j0-1)
  int po[NS], ro[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    po[s] = (row[s] + 2) * N + i;
    ro[s] = (row[s] + 1) * N + i;
  }
  // restriction epilogue (fine_kernel FM_PREX): thread (xI, xrow)
  constexpr int NCX = N / 2;
  const int xI = tid % NCX, xrow = tid / NCX;
  const bool xon = xrow < TY && xI >= 1;
  double xacc = 0.0;
  double* tout = a.t + (int64_t)mu * NCX * N * NCX + (int64_t)(j0 + xrow) * NCX + xI;
  auto xz = [&](int kk) {
    if (!xon) return;
    const double* R1 = rbuf + (kk & 1) * CSZ + xrow * N + 2 * xI;
    const double v = 0.5 * (R1[-1] + R1[1]) + R1[0];
    if (kk & 1) {
      xacc += 0.5 * v;
      const int K = (kk - 1) >> 1;
      if (K >= 1) tout[(int64_t)K * N * NCX] = xacc;
      xacc = 0.5 * v;
    } else {
      xacc += v;
    }
  };

  double pd[NS], pc[NS], pu[NS];  // p(k-1), p(k), p(k+1) of every slot
  double ud[2] = {0.0, 0.0}, uc[2] = {0.0, 0.0};  // u(k-2), u(k-1) of the own rows
  double rp[2] = {0.0, 0.0};                       // r_new(k-1) of the own rows
  double part[2] = {0.0, 0.0};
  double acc = 0.0;
  wait(0);
  wait(1);
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    pd[s] = ring[(0 % S) * STAGE + po[s]];
    pc[s] = ring[(1 % S) * STAGE + po[s]];
  }
  __syncthreads();  // plane 0's slot is free: the ring then holds planes k .. k+3 in iteration k
  if (tid == 0 && S <= N) issue(S);
  // running pointers of the own rows' x / r entries on the current plane (x is staged with the
  // plane: a dependent global load would stall every plane)
  double* xp[2];
  double* rq[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int64_t g = base + (int64_t)(j0 + row[s]) * N + i + N2;  // plane 1
    xp[s] = a.x + g;
    rq[s] = a.rout + g;
  }
  int xo[2];  // own rows inside the staged x rows
#pragma unroll
  for (int s = 0; s < 2; ++s) xo[s] = PSZ + RSZ + row[s] * N + i;

  // one plane of the CG update (math only): r_new and u = w D^-1 r_new of every slot
  auto cgmath = [&](int k, double* un, double* rn) {
    const double* SK = ring + (k % S) * STAGE;
    const double* SU = ring + ((k + 1) % S) * STAGE;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s == 2 && !has3) continue;
      pu[s] = SU[po[s]];
      const double* P = SK + po[s];
      const double offx = fma(wxm[s], P[-1], wxp[s] * P[1]);
      const double offy = fma(wym[s], P[-N], wyp[s] * P[N]);
      const double offz = fma(wzm[s], pd[s], wzp[s] * pu[s]);
      const double off = (offx + offy) + offz;
      const double Au = fma(dg[s], pc[s], -off);
      // (ghosts and rows outside the grid: exact zeros, whatever the unstaged rows hold)
      rn[s] = on[s] ? fma(-al, Au, SK[PSZ + ro[s]]) : 0.0;
      un[s] = on[s] ? wdi[s] * rn[s] : 0.0;
    }
  };
  // pre-smoothing residual of plane k-1 without its upper z face (weights of plane k-1)
  auto prepart = [&](int k) {
    const double* U = uring + ((k - 1) & 1) * USZ;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* P = U + ro[s];
      const double offx = fma(wxm[s], P[-1], wxp[s] * P[1]);
      const double offy = fma(wym[s], P[-N], wyp[s] * P[N]);
      part[s] = fma(1.0 - om, rp[s], (offx + offy) + wzm[s] * ud[s]);
    }
  };
  // results of plane k: u ring, x, r, and r1(k-1) finished with plane k's lower z face
  auto stores = [&](int k, const double* un, const double* rn) {
    const double* SK = ring + (k % S) * STAGE;
    double* UK = uring + (k & 1) * USZ;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s == 2 && !has3) continue;
      UK[ro[s]] = un[s];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (on[s]) {
        *xp[s] = fma(al, pc[s], SK[xo[s]]);
        *rq[s] = rn[s];
        acc = fma(rn[s], rn[s], acc);
      }
      xp[s] += N2;
      rq[s] += N2;
    }
    if (k >= 2) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
        rbuf[((k - 1) & 1) * CSZ + row[s] * N + i] = on[s] ? fma(wzm[s], un[s], part[s]) : 0.0;
    }
  };
  auto rotate = [&](const double* un, const double* rn) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      pd[s] = pc[s];
      pc[s] = pu[s];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      ud[s] = uc[s];
      uc[s] = un[s];
      rp[s] = rn[s];
    }
  };
  // (a split arrive / wait CTA barrier that lets the CG math of steady planes run ahead of the
  // wait measured slower: 2.26 vs 2.04 ms, profiles/r02g_cgp.md)
#pragma unroll kCgpUnroll
  for (int k = 1; k < N; ++k) {
    if (k >= 2) prepart(k);
    refresh(k);
    wait(k + 1);
    double un[NS], rn[NS];
    cgmath(k, un, rn);
    stores(k, un, rn);
    __syncthreads();  // u(k), r1(k-1) visible; plane k's ring slot is free
    if (tid == 0 && k + S <= N) issue(k + S);
    if (k >= 2) xz(k - 1);
    rotate(un, rn);
  }
  prepart(N);  // drain: r1(N-1) (u(N) = 0), with the weights of plane N-1
#pragma unroll
  for (int s = 0; s < 2; ++s)
    rbuf[((N - 1) & 1) * CSZ + row[s] * N + i] = on[s] ? part[s] : 0.0;
  __syncthreads();
  xz(N - 1);
  __shared__ double red[32];
  const double sred = block_reduce_sum(acc, red);
  if (tid == 0) {
    // the CG update kernel's partial geometry: this tile covers tiles / ytiles of its slots
    const int per = a.tiles / (N / TY);
    double* P = a.partial + (int64_t)mu * a.tiles + yt * per;
    P[0] = sred;
    for (int u = 1; u < per; ++u) P[u] = 0.0;
  }
}

}  // namespace

// rbws_set_kernel_variant(4, .) / RBWS_CGP: on where it applies (default), 0 = the separate
// CG update and pre-smoothing kernels
static std::atomic<int> g_cgp{[] {
  const char* e = getenv("RBWS_CGP");
  return (e && atoi(e) == 0) ? 0 : 1;
}()};
int fine_set_cgp(int v) {
  if (v < -1 || v > 1) return 1;
  g_cgp.store(v == 0 ? 0 : 1);
  return 0;
}
int fine_cgp_variant() { return g_cgp.load(); }

template <int N>
static bool cgp_fits(const Sep7& op, int batch) {
  const FineGeom g = fine_geom(op.n, batch);  // the CG update kernel's partial slots
  if (g.tiles % (N / CgpGeom<N>::TY)) return false;
  // whole z-range per CTA: enough CTAs to fill the GPU
  if ((int64_t)batch * (N / CgpGeom<N>::TY) < 148) return false;
  return CgpGeom<N>::bytes(op.Q) <= 227 * 1024;
}

bool fine_cgp_ok(const Sep7& op, int batch, const LaunchCtx& lc) {
  if (!g_cgp.load(std::memory_order_relaxed) || op.wface || lc.zhi > 0) return false;
  if (op.n == 64) return cgp_fits<64>(op, batch);
  if (op.n == 128) return cgp_fits<128>(op, batch);
  return false;
}

template <int N>
static cudaError_t cgp_launch(const CgpArgs& a, int batch, cudaStream_t stream) {
  const size_t smem = CgpGeom<N>::bytes(a.op.Q);
  cudaError_t e = smem_attr((const void*)cgp_kernel<N>, smem);
  if (e != cudaSuccess) return e;
  dim3 grd(1, N / CgpGeom<N>::TY, batch);
  count_launch();
  cgp_kernel<N><<<grd, kCgpThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t fine_cg_update_pre(const Sep7& op, int batch, const double* p, double* x,
                               const double* r_in, double* r_out, const double* alpha,
                               double* partial, double* t, double omega, const LaunchCtx& lc) {
  if (r_in == r_out) return cudaErrorInvalidValue;
  if (!fine_cgp_ok(op, batch, lc)) return cudaErrorInvalidValue;
  CgpArgs a{};
  a.op = op;
  a.p = p;
  a.x = x;
  a.rin = r_in;
  a.rout = r_out;
  a.t = t;
  a.alpha = alpha;
  a.partial = partial;
  a.tiles = fine_geom(op.n, batch).tiles;
  a.active = lc.active;
  a.omega = omega;
  return op.n == 64 ? cgp_launch<64>(a, batch, lc.stream) : cgp_launch<128>(a, batch, lc.stream);
}

}  // namespace rbws
