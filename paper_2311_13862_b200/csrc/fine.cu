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
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include "fine.cuh"
#include "tma.cuh"

namespace rbws {

constexpr int kStages = 8;  // ring slots (power of two)
constexpr int kMaxKz = 64;  // planes per z-chunk (bounds the z-factor table)
constexpr int kMaxDiagChanges = 16;  // DC kernels when the diagonal changes on <= 16 planes

// test/A-B override of the DC choice (rbws_set_kernel_variant): -1 auto, 0 never, 1 whenever
// the diagonal changes on few enough planes (any N)
static std::atomic<int> g_force_dc{[] {
  const char* e = getenv("RBWS_DC");  // A/B runs: "0" never, "1" whenever applicable
  return e ? atoi(e) : -1;
}()};
int fine_set_dc(int v) {
  if (v < -1 || v > 1) return 1;
  g_force_dc.store(v);
  return 0;
}
// SW ("scaled weights") pre-smoothing kernels: -1 auto (whenever the diagonal changes on few
// planes and the weights are not stored), 0 never, 1 = auto
static std::atomic<int> g_force_sw{[] {
  const char* e = getenv("RBWS_PRE_SW");
  return e ? atoi(e) : -1;
}()};
int fine_set_sw(int v) {
  if (v < -1 || v > 1) return 1;
  g_force_sw.store(v);
  return 0;
}
// p-update kernel without the transformed ring (the neighbours' p = s + beta p_old formed
// where they are read; 80 registers, three CTAs per SM; bitwise the transformed-ring kernel):
// opt-in (RBWS_PAPPLY_DIRECT=1 / rbws_set_kernel_variant(3, 1)) — measured slower on configs[1],
// 1.12 -> 1.17 ms per full launch (1.24 ms at two CTAs per SM): unlike the pre-smoothing it
// saves no HBM stream, and the 8 neighbour loads + 4 FMAs per node cost more than the
// transformed ring's store + barrier coupling
static std::atomic<int> g_direct_papply{[] {
  const char* e = getenv("RBWS_PAPPLY_DIRECT");
  return (e && atoi(e) == 1) ? 1 : 0;
}()};
int fine_set_direct(int v) {
  if (v < -1 || v > 1) return 1;
  g_direct_papply.store(v == 1 ? 1 : 0);
  return 0;
}
int fine_variant() {
  return (g_force_dc.load() + 1) + 4 * (g_force_sw.load() + 1) + 16 * g_direct_papply.load();
}
constexpr int kThreads = 256;  // threads per CTA (one per grid column of the tile; N = 512: 512)

// Compile-time tile geometry for a grid with N cells per axis: RPP rows per pass
// of the CTA, NPT rows per thread, TY = RPP*NPT rows per tile.  All shared-memory
// and global offsets below are compile-time multiples of N, so a neighbour read
// is one LDS with an immediate offset from a per-plane base register.
#ifndef RBWS_N512_NPT
#define RBWS_N512_NPT 2
#endif
#ifndef RBWS_SMALL_NPT
#define RBWS_SMALL_NPT 2
#endif
template <int N, int T = kThreads>
struct FT {
  static constexpr int RPP = (T / N) < 1 ? 1 : ((T / N) < N ? T / N : N);
  static constexpr int NPT = N >= 512 ? RBWS_N512_NPT : ((RPP * 2 <= N) ? RBWS_SMALL_NPT : 1);
  static constexpr int TY = RPP * NPT;
  static constexpr int THREADS = RPP * N;
  static constexpr int HSZ = (TY + 2) * N;  // doubles per staged array with halo rows
  static constexpr int CSZ = TY * N;        // doubles per staged array, tile rows only
};

// threads per CTA of a mode: the prolongation + post-smoothing kernel runs 512-thread
// CTAs (16-row tiles) at N = 64: half the halo-row work per node, measured -5 %
int fine_mode_threads(int mode, int n) {
#ifndef RBWS_PREX_512
#define RBWS_PREX_512 0
#endif
  if (RBWS_PREX_512 && mode == 7 && n == 64) return 512;
  return (mode == 6 && (n == 64 || n == 128)) ? 512 : kThreads;
}

FineGeom fine_geom(int n, int batch, int nz, int threads) {
  FineGeom g;
  if (threads <= 0) threads = kThreads;
  int rpp = threads / n;
  if (rpp < 1) rpp = 1;
  if (rpp > n) rpp = n;
  g.rpp = rpp;
  g.npt = n >= 512 ? RBWS_N512_NPT : ((rpp * 2 <= n) ? RBWS_SMALL_NPT : 1);
  g.ty = rpp * g.npt;
  g.threads = rpp * n;
  g.ytiles = n / g.ty;
  if (nz <= 0) nz = n;
  g.zc = 1;
  while ((nz + g.zc - 1) / g.zc > kMaxKz) g.zc *= 2;
  while ((int64_t)g.ytiles * batch * g.zc < 2 * 148 && (nz / (g.zc * 2)) >= 8) g.zc *= 2;
  g.kz = (nz + g.zc - 1) / g.zc;
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
  int zlo, zhi;   // output planes [zlo, zhi) (global plane indices, virtual base pointers)
  int dc;         // PRE / POSTP: w/diag from the cached shared-memory tile (h1 unused)
  int sw;         // PRE / PREX: scaled weights on the raw b (h1 read on rebuild planes only)
  int c0_shared;  // c0 is one instance shared by the whole batch (e.g. the rhs f)
  const double* ec;  // FM_POSTP: coarse-grid correction (n/2 cells, padded batch layout)
};

enum FineMode : int {
  FM_APPLY = 0,   // h0 = x                  out0 = A x (optional), dot x.Ax
  FM_RESID = 1,   // h0 = x, c0 = b          out0 = b - A x, dot |r|^2
  FM_JACOBI = 2,  // h0 = x, c0 = b          out0 = x + w (b - A x)/d, dot b.out
  FM_PRE = 3,     // h0 = b, h1 = dinv       out0 = b - A (w dinv b)
  FM_CG = 4,      // h0 = p, c0 = x, c1 = r  x += a p, r -= a A p (in place), dot |r|^2
  FM_PAPPLY = 5,  // h0 = s, h1 = p_old      out0 = p = s + b p_old, dot p.Ap
  FM_POSTP = 6,   // h0 = b, h1 = dinv, ec   u = w dinv b + P ec; out0 = u + w (b - A u)/d, dot b.out
  FM_PREX = 7,    // h0 = b, h1 = dinv       r1 = b - A (w dinv b), restricted along x and z in the
                  //                         CTA: out0 = t[K][j][I] (n/2 x n x n/2 per instance)
};

// DC ("diagonal cached"): PRE / POSTP keep w/diag of the staged rows in a shared-memory
// tile, reloaded from the 1/diag vector only on planes where the diagonal changes along z
// (thermal blocks: a few planes), instead of streaming 1/diag with every plane (8 bytes
// per node less; bitwise the same values)
// tile geometry of a mode (see fine_mode_threads)
template <int MODE, int N>
using FTM = FT<N, ((MODE == FM_POSTP && (N == 64 || N == 128)) ||
                   (RBWS_PREX_512 && MODE == FM_PREX && N == 64)) ? 512 : kThreads>;

// SW ("scaled weights", FM_PRE / FM_PREX): the stencil of u = w D^-1 b is taken on the raw b
// with the face weights pre-multiplied by the neighbours' w/diag, cached in registers and
// rebuilt only on planes around a change of the z factors (1/diag read through L2 there):
// no transformed ring, no 1/diag stream
template <int MODE, int N, bool DC = false, bool SW = false>
struct SL {
  // PRE / PAPPLY stencil a derived vector (w dinv b, s + beta p_old): each staged
  // plane is transformed once into a second ring, so neighbours cost one LDS
  static constexpr bool XF = !SW && (MODE == FM_PRE || MODE == FM_PREX || MODE == FM_PAPPLY ||
                                     MODE == FM_POSTP);
  // SW on FM_PAPPLY ("direct"): no transformed ring either; the neighbours' p = s + beta p_old
  // are formed from the two staged arrays where they are read
  static constexpr bool DIRECT = SW && MODE == FM_PAPPLY;
  static constexpr int NH = (XF || DIRECT) ? 2 : 1;  // DC: h1 (1/diag) staged only on reload planes
  static constexpr int NC = (MODE == FM_CG) ? 2 : ((MODE == FM_RESID || MODE == FM_JACOBI) ? 1 : 0);
  // raw / transformed ring slots (N = 512 rows are 4 KB: a shallower raw ring fits 227 KB).
  // U >= 6: a trip reads transformed planes k-1 .. k+2 while the next trip's transform
  // (no barrier in between) writes k+3, k+4.
  // N = 256: rings shallow enough for two CTAs per SM (pre-smoothing / p-update 15.6 ->
  // 10.3 ms, CG update 16.2 -> 11.3 ms per launch on configs[3]; the post-smoothing kernel
  // fits two only without the z-factor table, i.e. with stored weights)
#ifndef RBWS_N256_XF_S
#define RBWS_N256_XF_S 3
#endif
#ifndef RBWS_N128_XF_S
#define RBWS_N128_XF_S 4
#endif
// raw ring slots of the 512-thread post-smoothing kernel at N = 128 (one CTA per SM)
#ifndef RBWS_N128_POSTP_S
#define RBWS_N128_POSTP_S 4
#endif
// residual kernel (initial and true residual of every solve) at N <= 64: CTAs per SM
#ifndef RBWS_RESID_CTAS
#define RBWS_RESID_CTAS 2
#endif
// raw ring slots of the scaled-weights kernels at N = 128 (4: three CTAs per SM fit)
#ifndef RBWS_N128_SW_S
#define RBWS_N128_SW_S 6
#endif
  static constexpr int S = XF ? (N >= 512 ? (RBWS_N512_NPT == 2 ? (MODE == FM_POSTP ? 2 : 3) : 4)
                                          : (N >= 256 ? (MODE == FM_POSTP ? 3 : RBWS_N256_XF_S)
                                                      : (N >= 128 ? (MODE == FM_PREX ? 3 : (MODE == FM_POSTP ? RBWS_N128_POSTP_S : RBWS_N128_XF_S))
                                                                  : 6)))
                              : (N >= 128 ? ((SW && N == 128) ? RBWS_N128_SW_S : 6)
                                          : ((DIRECT || (RBWS_RESID_CTAS == 3 && MODE == FM_RESID))
                                                 ? 6 : kStages));
  static constexpr int U = 6;
};

// FM_POSTP stages, with every even fine plane p, coarse plane p/2 + 1 rows
// [cj0, cj0 + CR) (cj0 = first coarse row the tile's rows j0-1 .. j0+TY touch)
template <int N, int TY_ = FT<N>::TY>
struct FCoarse {
  static constexpr int NCC = N / 2;
  static constexpr int CR = TY_ / 2 + 3;
  static constexpr int CSZ = CR * NCC;
};

#ifndef RBWS_MIN_CTAS
#define RBWS_MIN_CTAS 2
#endif

template <int N, int MODE, bool DC = false, bool SW = false>
struct FSmem {
  using L = SL<MODE, N, DC, SW>;
  using G = FTM<MODE, N>;
  static constexpr int STAGE = L::NH * G::HSZ + L::NC * G::CSZ +
                               (MODE == FM_POSTP ? FCoarse<N, G::TY>::CSZ : 0);
  // raw ring, transformed ring, cached w/diag tile (DC)
  static constexpr int RING = L::S * STAGE + (L::XF ? L::U * G::HSZ : 0) +
                              (DC ? G::HSZ : 0) + (MODE == FM_PREX ? 4 * G::CSZ : 0);
  static size_t bytes(int np, int Q) {
    return 64 + 4 * (kMaxKz + 4) + (SW ? 16 : 0) + 8 * (((size_t)np * 3 * Q + 1) & ~(size_t)1) +
           8 * (size_t)RING;
  }
};

// SCW ("stored coefficient weights"): the face weights come from per-instance arrays
// (Sep7::wface, built at batch setup) instead of registers refreshed from the separable
// tables — for coefficients whose z factors change on most planes, where the refresh
// (5Q terms per node and plane) dominates; bitwise the same weights
// SW kernels at N <= 128: 80 registers without spills, three CTAs per SM (pre-smoothing
// 0.86 -> 0.81 ms per full configs[1] launch)
#ifndef RBWS_SW_MIN_CTAS
#define RBWS_SW_MIN_CTAS 3
#endif
template <int MODE, int N, bool DC, bool SCW, bool SW = false>
__global__ void __launch_bounds__(FTM<MODE, N>::THREADS,
                                  FTM<MODE, N>::THREADS <= 256
                                      ? ((SW && N <= 128) ? RBWS_SW_MIN_CTAS
                                         : ((MODE == FM_RESID && N <= 64 && !SCW) ? RBWS_RESID_CTAS
                                                                                   : RBWS_MIN_CTAS))
                                      : 1)
fine_kernel(FineArgs a) {
  static_assert(!SW || ((MODE == FM_PRE || MODE == FM_PREX || MODE == FM_PAPPLY) && !DC && !SCW),
                "SW: PRE / PREX (scaled weights) and PAPPLY (direct neighbours) only");
  constexpr bool SCALED = SW && (MODE == FM_PRE || MODE == FM_PREX);
  constexpr bool DIRECT = SW && MODE == FM_PAPPLY;
  using G = FTM<MODE, N>;
  using L = SL<MODE, N, DC, SW>;
  constexpr bool XF = L::XF;
  constexpr int NH = L::NH, NC = L::NC, S = L::S, U = L::U;
  constexpr int NPT = G::NPT, RPP = G::RPP, TY = G::TY;
  constexpr int HSZ = G::HSZ, CSZ = G::CSZ;
  constexpr int STAGE = FSmem<N, MODE, DC, SW>::STAGE;  // doubles per raw ring slot
  constexpr int64_t N2 = (int64_t)N * N;
  extern __shared__ __align__(128) unsigned char smem[];
  const Sep7& op = a.op;
  const int Q = op.Q, ZW = SCW ? 0 : 3 * Q;  // SCW: no z-factor table (weights are stored)
  const int zc = a.g.zc;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (a.active && !a.active[mu]) return;
  const int yt = blockIdx.y;
  const int j0 = yt * TY;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)mu * N2 * N;
  const int kz = a.g.kz;
  const int kb0 = max(1, a.zlo + kc * kz), ke = min(min(N, a.zhi), a.zlo + (kc + 1) * kz);
  // FM_PREX on a z-chunk starting at an even plane 2K: coarse plane K also needs fine plane
  // 2K-1, so the chunk recomputes it (output planes from kb0 - 1; nothing is written for it)
  const int kb = (MODE == FM_PREX && kb0 > 1) ? kb0 - 1 : kb0;
  if (kb >= ke) {  // empty chunk (never for the geometries fine_geom builds)
    if (a.dot != DOT_NONE && tid == 0) a.partial[(int64_t)mu * a.g.tiles + yt * zc + kc] = 0.0;
    return;
  }
  const int p_first = kb - 1, p_last = ke;  // staged planes (inclusive)
  const int np = p_last - p_first + 1;

  // ---- shared memory carve-up (offsets multiples of 16 bytes)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);            // [S]
  int* zsame = reinterpret_cast<int*>(smem + 64);                // [kMaxKz + 2]
  uint32_t* swbits = reinterpret_cast<uint32_t*>(smem + 64 + 4 * (kMaxKz + 4));  // [4] (SW)
  double* zf = reinterpret_cast<double*>(smem + 64 + 4 * (kMaxKz + 4) + (SW ? 16 : 0));  // [np][3Q]
  double* ring = zf + ((np * ZW + 1) & ~1);                      // [S][STAGE]
  double* uring = ring + S * STAGE;                              // [U][HSZ] (XF)
  double* wd = uring + (XF ? U * HSZ : 0);                       // [HSZ] w/diag (DC)
  double* rbuf = wd + (DC ? HSZ : 0);  // FM_PREX: r1 of [2 trips][2 planes][TY rows][N]

  for (int t = tid; t < np * ZW; t += G::THREADS) {  // z factors of the staged planes
    const int p = t / (3 * Q), f = (t / Q) % 3, q = t % Q, k = p_first + p;
    const double* F = op.face + (size_t)q * 3 * N;
    const double* NF = op.node + (size_t)q * 9 * (N + 1);
    double v;
    if (f == 0) v = NF[(0 * 3 + 2) * (N + 1) + k];       // x-part along z
    else if (f == 1) v = NF[(1 * 3 + 2) * (N + 1) + k];  // y-part along z
    else v = (k < N) ? F[2 * N + k] : 0.0;               // z-face k, k+1
    zf[t] = v;
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  if (SCALED && tid < 64) {  // plane flags of the staged planes, 32 per word
    const int m = p_first + tid;
    const bool f = tid < np && (m <= 1 || m >= N || __ldg(op.fz + m) != 0);
    const uint32_t bits = __ballot_sync(0xffffffffu, f);
    if ((tid & 31) == 0) swbits[tid >> 5] = bits;
  }
  __syncthreads();
  for (int p = 1 + tid; p < np; p += G::THREADS) {  // plane p repeats plane p-1's z factors?
    int same = 1;
    for (int t = 0; t < ZW; ++t) same &= (zf[p * ZW + t] == zf[(p - 1) * ZW + t]);
    zsame[p] = same;
  }

  const int skip = (j0 == 0) ? 1 : 0;  // row j0-1 does not exist for the first tile
  constexpr int NCC = FCoarse<N, TY>::NCC;
  const int cj0 = (j0 == 0) ? 0 : (j0 >> 1) - 1;  // first staged coarse row (FM_POSTP)
  auto issue = [&](int p) {
    const int sl = (p - p_first) % S;
    double* st = ring + sl * STAGE;
    const uint32_t hbytes = (uint32_t)((TY + 2 - skip) * N * 8);
    constexpr uint32_t cbytes = (uint32_t)(CSZ * 8);
    constexpr uint32_t ebytes = (uint32_t)(FCoarse<N, TY>::CSZ * 8);
    // coarse plane p/2 + 1 (for the z march of P ec) with every even fine plane;
    // none past the last coarse plane (its ghost plane p/2 = n/2 is never advanced from)
    const bool stage_c = (MODE == FM_POSTP) && !(p & 1) && ((p >> 1) + 1 <= NCC);
    const bool h1_on = !DC || p == p_first || !__ldg(op.fz + p);  // DC: reload planes only
    mbar_arrive_expect_tx(&bar[sl], (NH > 1 && !h1_on ? 1 : NH) * hbytes + NC * cbytes +
                                        (stage_c ? ebytes : 0u));
    const int64_t plane = base + (int64_t)p * N2;
    const int64_t hrow = plane + (int64_t)(j0 - 1 + skip) * N;
    bulk_g2s(st + skip * N, a.h0 + hrow, hbytes, &bar[sl]);
    if (NH > 1 && h1_on) bulk_g2s(st + HSZ + skip * N, a.h1 + hrow, hbytes, &bar[sl]);
    if (NC > 0)
      bulk_g2s(st + NH * HSZ, a.c0 + (a.c0_shared ? plane - base : plane) + (int64_t)j0 * N,
               cbytes, &bar[sl]);
    if (NC > 1) bulk_g2s(st + NH * HSZ + CSZ, a.c1 + plane + (int64_t)j0 * N, cbytes, &bar[sl]);
    if (stage_c) {
      const int64_t cpl = (int64_t)mu * NCC * NCC * NCC + (int64_t)((p >> 1) + 1) * NCC * NCC +
                          (int64_t)cj0 * NCC;
      bulk_g2s(st + NH * HSZ, a.ec + cpl, ebytes, &bar[sl]);
    }
  };
  auto wait = [&](int p) {
    const int t = p - p_first;
    mbar_wait(&bar[t % S], (uint32_t)((t / S) & 1));
  };
  auto raw = [&](int p) -> const double* { return ring + ((p - p_first) % S) * STAGE; };
  if (tid == 0)
    for (int p = p_first; p <= p_last && p < p_first + S; ++p) issue(p);
  __syncthreads();  // zsame flags visible
  // bit p - p_first of zmask: plane p repeats plane p-1's z factors (np <= 66 planes)
  uint64_t zmask = 0;
  for (int p = 1; p < np && p < 64; ++p) zmask |= (uint64_t)(zsame[p] != 0) << p;
  const bool zlast = (np > 64) ? zsame[64] != 0 : false;  // kz = 64: plane p_first + 64 = ke - 1
  auto repeats = [&](int k) -> bool {  // CTA-uniform
    const int t = k - p_first;
    return t < 64 ? ((zmask >> t) & 1) != 0 : (MODE == FM_PREX ? zsame[t] != 0 : zlast);
  };
  // SW: plane k keeps plane k-1's scaled weights when the planes k-1, k, k+1 all repeat their
  // predecessor's face weights and diagonal (host-built flags op.fz; the Dirichlet planes 0
  // and n multiply zeros of b, so they never force a rebuild); bit t = plane p_first + t
  uint64_t smask = 0;
  auto fzx = [&](int m) -> bool { return m <= 1 || m >= N || __ldg(op.fz + m) != 0; };
  if (SCALED) {
    const uint64_t fm = ((uint64_t)swbits[1] << 32) | swbits[0];  // bit t: fzx(p_first + t)
    smask = (fm << 1) & fm & (fm >> 1);
  }
  auto steady_sw = [&](int k) -> bool {  // CTA-uniform
    const int t = k - p_first;
    if (t < 63) return ((smask >> t) & 1) != 0;
    return fzx(k - 1) && fzx(k) && fzx(k + 1);
  };

  // ---- this thread's column i and rows j = j0 + rl0 + r*RPP
  const int i = tid % N;
  const int rl0 = tid / N;
  const int hoff = (rl0 + 1) * N + i;  // thread's centre in a halo-staged array
  const int coff = rl0 * N + i;        // ... in a tile-only array
  bool on[NPT];
#pragma unroll
  for (int r = 0; r < NPT; ++r) on[r] = (i != 0) && (j0 + rl0 + r * RPP != 0);  // Dirichlet ghosts
  const double* th = op.theta + (size_t)mu * Q;
  const double sc = a.scal ? a.scal[mu] : 0.0;
  const double om = a.omega;
  double acc = 0.0;
  // cached face weights per owned row (recomputed only when the z factors change)
  double wxp[NPT] = {}, wxm[NPT] = {}, wyp[NPT] = {}, wym[NPT] = {}, wzp[NPT] = {}, wzm[NPT] = {};
  double dg[NPT] = {}, wdi[NPT] = {};
  auto weights = [&](int r, const double* zk) {
    const int j = j0 + rl0 + r * RPP;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    if (i >= 1 && j >= 1) {
#pragma unroll 2
      for (int q = 0; q < Q; ++q) {
        const double* F = op.face + (size_t)q * 3 * N;
        const double* NF = op.node + (size_t)q * 9 * (N + 1);
        const double t = th[q];
        const double tx = t * __ldg(NF + (0 * 3 + 1) * (N + 1) + j) * zk[q];       // theta N_xy(j) zx(k)
        const double tyv = t * __ldg(NF + (1 * 3 + 0) * (N + 1) + i) * zk[Q + q];  // theta N_yx(i) zy(k)
        const double tz = t * __ldg(NF + (2 * 3 + 0) * (N + 1) + i) * __ldg(NF + (2 * 3 + 1) * (N + 1) + j);
        a0 = fma(__ldg(F + 0 * N + i), tx, a0);
        a1 = fma(__ldg(F + 0 * N + i - 1), tx, a1);
        a2 = fma(__ldg(F + 1 * N + j), tyv, a2);
        a3 = fma(__ldg(F + 1 * N + j - 1), tyv, a3);
        a4 = fma(tz, zk[2 * Q + q], a4);
      }
    }
    wxp[r] = a0; wxm[r] = a1; wyp[r] = a2; wym[r] = a3; wzp[r] = a4;
  };
  auto diag = [&](int r) {
    dg[r] = ((wxp[r] + wxm[r]) + (wyp[r] + wym[r])) + (wzp[r] + wzm[r]);
    wdi[r] = om / dg[r];  // cached damping / diagonal (no per-node division)
  };
  // SW: face weights of node (i, j, k) times w/diag of the neighbour across the face (a.h1 =
  // 1/diag, read through L2 on the few planes where the weights are rebuilt)
  auto scaled = [&](int r, int k, int64_t gidx) {
    weights(r, zf + (k - p_first) * ZW);  // wxp, wxm, wyp, wym, wzp of plane k
    double zm = 0.0;                      // z face (k-1, k): the z weight of plane k-1
    const int j = j0 + rl0 + r * RPP;
    if (i >= 1 && j >= 1) {
      const double* zk = zf + (k - 1 - p_first) * ZW;
#pragma unroll 2
      for (int q = 0; q < Q; ++q) {
        const double* NF = op.node + (size_t)q * 9 * (N + 1);
        const double tz = th[q] * __ldg(NF + (2 * 3 + 0) * (N + 1) + i) * __ldg(NF + (2 * 3 + 1) * (N + 1) + j);
        zm = fma(tz, zk[2 * Q + q], zm);
      }
    }
    const double* D = a.h1 + gidx;
    wxp[r] *= om * __ldg(D + 1);
    wxm[r] *= om * __ldg(D - 1);
    wyp[r] *= om * __ldg(D + N);
    wym[r] *= om * __ldg(D - N);
    // (planes 0 and n hold zeros of b: their factor only has to be the one a steady plane
    // above / below would use)
    wzp[r] *= om * __ldg(k + 1 < N ? D + N2 : D);
    wzm[r] = zm * (om * __ldg(k > 1 ? D - N2 : D));
  };
#pragma unroll
  for (int r = 0; r < NPT; ++r) {  // plane kb-1: its z face (kb-1, kb) is wzm of plane kb
    if (SCW || SCALED) break;
    weights(r, zf);
    wzm[r] = wzp[r];
  }
  bool pend = false;  // wzm must take the previous plane's wzp on the next repeated plane

  // FM_POSTP: xy-interpolated coarse correction of every transformed row at coarse
  // planes K = p/2 and K+1 (rows: NPT own, then the halo rows j0-1 and j0+TY)
  double cv0[NPT + 2], cv1[NPT + 2];
  auto trow_j = [&](int t) { return t < NPT ? j0 + rl0 + t * RPP : (t == NPT ? j0 - 1 : j0 + TY); };
  auto trow_e = [&](int t) { return t < NPT ? hoff + t * RPP * N : (t == NPT ? i : (TY + 1) * N + i); };
  auto trow_on = [&](int t) { return t < NPT || (t == NPT ? (rl0 == 0 && !skip) : (rl0 == RPP - 1)); };
  const double hx = (i & 1) ? 0.5 : 0.0;
  // trilinear prolongation in x, y from a coarse plane C whose first row is crow0
  auto vxy = [&](const double* C, int crow0, int j) -> double {
    const double hy = (j & 1) ? 0.5 : 0.0;
    const double* q = C + ((j >> 1) - crow0) * NCC + (i >> 1);
    const double r0 = fma(hx, q[1] - q[0], q[0]);
    const double r1 = fma(hx, q[NCC + 1] - q[NCC], q[NCC]);
    return fma(hy, r1 - r0, r0);
  };
  if (MODE == FM_POSTP) {
    const double* E = a.ec + (int64_t)mu * NCC * NCC * NCC + (int64_t)(p_first >> 1) * NCC * NCC;
#pragma unroll
    for (int t = 0; t < NPT + 2; ++t)
      if (trow_on(t)) {
        cv0[t] = vxy(E, 0, trow_j(t));
        cv1[t] = vxy(E + NCC * NCC, 0, trow_j(t));
      }
  }
  // DC: w/diag of the staged rows, in shared memory; element e is only ever transformed by
  // one thread, so each thread refreshes its own elements from the staged 1/diag rows (h1,
  // bulk-copied only with the planes where the diagonal changes; host-built flags) and no
  // barrier is needed
  // XF: transform staged plane p (h0, h1) into the u ring; own rows returned in xo / bo
  auto transform = [&](int p, double* xo, double* bo) {
    const bool reload = DC && (p == p_first || !__ldg(op.fz + p));  // CTA-uniform
    const double* R = raw(p);
    double* T = uring + (p - p_first) % U * HSZ;
    const bool adv = (MODE == FM_POSTP) && p != p_first && !(p & 1);
    // three passes (coarse-plane advance, raw loads, stores): the compiler keeps shared-memory
    // loads behind earlier shared-memory stores, so row by row every row would wait for the
    // previous row's whole load -> FMA -> store chain
    if (adv) {
#pragma unroll
      for (int t = 0; t < NPT + 2; ++t) {
        if (!trow_on(t)) continue;
        cv0[t] = cv1[t];
        cv1[t] = vxy(R + NH * HSZ, cj0, trow_j(t));
      }
    }
    double rb[NPT + 2], rd[NPT + 2];
#pragma unroll
    for (int t = 0; t < NPT + 2; ++t) {
      if (!trow_on(t)) continue;
      const int e = trow_e(t);
      rb[t] = R[e];
      rd[t] = (DC && !reload) ? wd[e] : R[HSZ + e];
    }
#pragma unroll
    for (int t = 0; t < NPT + 2; ++t) {
      if (!trow_on(t)) continue;
      const int e = trow_e(t);
      double v;
      if (DC && reload) wd[e] = rd[t] = om * rd[t];  // staged with this plane
      if (MODE == FM_PRE || MODE == FM_PREX) {
        v = (DC ? rd[t] : om * rd[t]) * rb[t];  // w dinv b
      } else if (MODE == FM_PAPPLY) {
        v = fma(sc, rd[t], rb[t]);  // s + beta p_old
      } else {  // FM_POSTP: w dinv b + P ec
        const double pe = (p & 1) ? 0.5 * (cv0[t] + cv1[t]) : cv0[t];
        v = fma(DC ? rd[t] : om * rd[t], rb[t], pe);
      }
      T[e] = v;
      if (t < NPT) {
        xo[t] = v;
        bo[t] = rb[t];
      }
    }
  };

  // own-column stencil input of row r on staged plane p (non-transformed modes; DIRECT:
  // p = s + beta p_old formed here)
  auto own = [&](int p, int r) -> double {
    const double* R = raw(p) + hoff + r * RPP * N;
    return DIRECT ? fma(sc, R[HSZ], R[0]) : R[0];
  };
  // Own-column values march in registers: xd = u(k-1), xc = u(k); only the four
  // in-plane neighbours are read from shared memory.
  double xd[NPT], xc[NPT], bcv[NPT];
  if (XF) {
    wait(p_first);
    wait(p_first + 1);
    transform(p_first, xd, bcv);
    transform(p_first + 1, xc, bcv);
    __syncthreads();
    if (tid == 0) {
      if (p_first + S <= p_last) issue(p_first + S);
      if (p_first + 1 + S <= p_last) issue(p_first + 1 + S);
    }
  } else {
    wait(p_first);
    wait(p_first + 1);
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      xd[r] = own(p_first, r);
      xc[r] = own(p_first + 1, r);
    }
  }

  // one plane: vd / vc / vu = own-column input at k-1 / k / k+1, vb = own b at k
  int64_t gk = base + (int64_t)(j0 + rl0) * N + i + (int64_t)kb * N2;  // (i, j0+rl0, k)
  // face weights for plane k (refreshed only where the z factors change; CTA-uniform)
  auto refresh = [&](int k) {
    if (SCW) return;
    if constexpr (SCALED) {
      if (k == kb || !steady_sw(k)) {
#pragma unroll
        for (int r = 0; r < NPT; ++r) scaled(r, k, gk + r * RPP * N);
      }
      return;
    }
    if (k == kb || !repeats(k)) {
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        const double prev = wzp[r];
        weights(r, zf + (k - p_first) * ZW);
        wzm[r] = prev;
        diag(r);
      }
      pend = true;
    } else if (pend) {
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        wzm[r] = wzp[r];
        diag(r);
      }
      pend = false;
    }
  };
  // true when plane k keeps the current weights (no refresh work)
  auto steady = [&](int k) { return SCW || (k != kb && repeats(k) && !pend); };
  // SCW: stored weights; wzs[r] = z-face weight below the current node (previous plane)
  const double* WX = op.wface;
  const double* WY = op.wface + op.wstride;
  const double* WZ = op.wface + 2 * op.wstride;
  double wzs[NPT];
#pragma unroll
  for (int r = 0; r < NPT; ++r)
    wzs[r] = SCW ? __ldg(WZ + base + (int64_t)(j0 + rl0 + r * RPP) * N + i + (int64_t)(kb - 1) * N2)
                 : 0.0;
  // the NPT nodes of one plane: vd / vc / vu = own-column input at k-1 / k / k+1, vb = own b
  // the four in-plane neighbours of row r's node on plane k (shared memory)
  auto nbrs = [&](int k, int r, double* nb) {
    const double* P0 = (XF ? uring + (k - p_first) % U * HSZ : raw(k)) + hoff + r * RPP * N;
    if (DIRECT) {  // s + beta p_old of the neighbours
      nb[0] = fma(sc, P0[HSZ + 1], P0[1]);
      nb[1] = fma(sc, P0[HSZ - 1], P0[-1]);
      nb[2] = fma(sc, P0[HSZ + N], P0[N]);
      nb[3] = fma(sc, P0[HSZ - N], P0[-N]);
      return;
    }
    nb[0] = P0[1];
    nb[1] = P0[-1];
    nb[2] = P0[N];
    nb[3] = P0[-N];
  };
  auto node = [&](int k, int r, int64_t gk_, double ud, double uc, double uu, double vbr,
                  const double* nb) {
    const double* C0 = raw(k) + NH * HSZ + coff;
    const int o = r * RPP * N;  // compile-time after unrolling
    const double ue = nb[0], uw = nb[1], un = nb[2], us = nb[3];
    const int64_t gidx = gk_ + o;
    double xp, xm, yp, ym, zp, zm, dgr, wdr;
    if constexpr (SCW) {
      xp = __ldg(WX + gidx);
      xm = __ldg(WX + gidx - 1);
      yp = __ldg(WY + gidx);
      ym = __ldg(WY + gidx - N);
      zp = __ldg(WZ + gidx);
      zm = wzs[r];
      wzs[r] = zp;
      dgr = ((xp + xm) + (yp + ym)) + (zp + zm);
      // post-smoothing: w/diag from the staged 1/diag (no per-node division)
      // (the raw ring slot of plane k may already be refilled: read 1/diag through L2)
      wdr = (MODE == FM_POSTP) ? om * __ldg(a.h1 + gidx) : (MODE == FM_JACOBI ? om / dgr : 0.0);
    } else {
      xp = wxp[r]; xm = wxm[r]; yp = wyp[r]; ym = wym[r]; zp = wzp[r]; zm = wzm[r];
      dgr = dg[r];
      wdr = wdi[r];
    }
    // shallow FMA tree (a dependent chain of 6 would be latency bound)
    // (SW: the weights are scaled by the neighbours' w/diag and the input is b itself)
    if (SCALED) vbr = uc;
    const double offx = fma(xm, uw, xp * ue);
    const double offy = fma(ym, us, yp * un);
    const double offz = fma(zm, ud, zp * uu);
    const double off = (offx + offy) + offz;
    if (MODE == FM_PRE) {
      // b - A (w D^-1 b) = (1 - w) b + off(w D^-1 b): the diagonal term is w b
      if (on[r]) a.out0[gidx] = fma(1.0 - om, vbr, off);
    } else if (MODE == FM_PREX) {  // to the CTA's r1 buffer (ghost nodes: 0)
      const int t = k - kb;
      rbuf[(((t >> 1) & 1) * 2 + (t & 1)) * CSZ + coff + o] = on[r] ? fma(1.0 - om, vbr, off) : 0.0;
    } else if (MODE == FM_POSTP) {
      const double Au = fma(dgr, uc, -off);
      const double y = fma(wdr, vbr - Au, uc);
      if (on[r]) a.out0[gidx] = y;
      acc = on[r] ? fma(vbr, y, acc) : acc;
    } else {
      const double Au = fma(dgr, uc, -off);
      if (MODE == FM_APPLY) {
        if (on[r] && a.out0) a.out0[gidx] = Au;
        acc = on[r] ? fma(uc, Au, acc) : acc;
      } else if (MODE == FM_RESID) {
        const double rv = C0[o] - Au;
        if (on[r] && a.out0) a.out0[gidx] = rv;  // null: the norm only (true residual)
        acc = on[r] ? fma(rv, rv, acc) : acc;
      } else if (MODE == FM_JACOBI) {
        const double bv = C0[o];
        const double y = fma(wdr, bv - Au, uc);
        if (on[r]) a.out0[gidx] = y;
        acc = on[r] ? fma(bv, y, acc) : acc;
      } else if (MODE == FM_CG) {
        const double xv = fma(sc, uc, C0[o]);
        const double rv = fma(-sc, Au, C0[CSZ + o]);
        if (on[r]) {
          a.out0[gidx] = xv;
          a.out1[gidx] = rv;
        }
        acc = on[r] ? fma(rv, rv, acc) : acc;
      } else {  // FM_PAPPLY
        if (on[r]) a.out0[gidx] = uc;
        acc = on[r] ? fma(uc, Au, acc) : acc;
      }
    }
  };
  auto step = [&](int k, const double* vd, const double* vc, const double* vu, const double* vb) {
    refresh(k);
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      double nb[4];
      nbrs(k, r, nb);
      node(k, r, gk, vd[r], vc[r], vu[r], vb[r], nb);
    }
    gk += N2;
  };

  // FM_PREX epilogue: thread (I, orow) restricts row j0+orow of plane kk along x
  // (0.5 r(2I-1) + r(2I) + 0.5 r(2I+1), the order of restrict_kernel) and accumulates the
  // z weights 0.5 / 1 / 0.5 of coarse plane K in a register; a completed coarse plane goes
  // to t[K][j][I].  Needs the whole z-range of the instance in one CTA (zc == 1).
  constexpr int NCX = N / 2;
  const int xI = tid % NCX, xrow = tid / NCX;
  const bool xon = (MODE == FM_PREX) && xrow < TY && xI >= 1;
  double xacc = 0.0;
  double* tout = a.out0 + (int64_t)mu * NCX * N * NCX + (int64_t)(j0 + xrow) * NCX + xI;
  auto xload = [&](int kk) -> double {  // x-restricted r1 of plane kk at (xI, xrow)
    const int t = kk - kb;
    const double* R1 = rbuf + (((t >> 1) & 1) * 2 + (t & 1)) * CSZ + xrow * N + 2 * xI;
    return 0.5 * (R1[-1] + R1[1]) + R1[0];
  };
  auto xz = [&](int kk, double v) {
    if (!xon) return;
    if (kk & 1) {  // 2K+1: closes coarse plane K (if 2K-1 was in this chunk), opens K+1
      xacc += 0.5 * v;
      const int K = (kk - 1) >> 1;
      if (K >= 1 && kk >= kb + 2) tout[(int64_t)K * N * NCX] = xacc;
      xacc = 0.5 * v;
    } else {
      xacc += v;
    }
  };

  // two planes per trip with statically rotating register roles: one CTA barrier
  // and two TMA issues amortised over two nodes per row
  for (int k0 = kb; k0 < ke; k0 += 2) {
    double u0[NPT], u1[NPT], b0[NPT], b1[NPT];
    const bool two = k0 + 1 < ke;
    if (XF) {
      wait(k0 + 1);
      transform(k0 + 1, u0, b0);
      if (k0 + 2 <= p_last) {
        wait(k0 + 2);
        transform(k0 + 2, u1, b1);
      }
      __syncthreads();  // transformed planes visible; raw slots of k0+1, k0+2 free
      if (tid == 0) {
        if (k0 + 1 + S <= p_last) issue(k0 + 1 + S);
        if (k0 + 2 + S <= p_last) issue(k0 + 2 + S);
      }
      if (MODE == FM_PREX && k0 > kb && xon) {  // the previous trip's r1 planes are complete
        const double v0 = xload(k0 - 2), v1 = xload(k0 - 1);
        xz(k0 - 2, v0);
        xz(k0 - 1, v1);
      }
    } else {
      wait(k0 + 1);
#pragma unroll
      for (int r = 0; r < NPT; ++r) u0[r] = own(k0 + 1, r);
      if (two) {
        wait(k0 + 2);
#pragma unroll
        for (int r = 0; r < NPT; ++r) u1[r] = own(k0 + 2, r);
      }
    }
    if (two && (SCALED ? (k0 != kb && steady_sw(k0) && steady_sw(k0 + 1))
                   : (steady(k0) && repeats(k0 + 1)))) {
      // common case: both planes keep the weights; one straight-line block of 2*NPT
      // independent nodes (latency hiding by ILP)
      // (all neighbour loads first: FM_PREX stores r1 to shared memory, which the compiler
      // must otherwise keep ordered with the next node's loads)
      // (measured: FM_PREX 1.35 -> 1.29 ms, SW 1.23 -> 0.87 ms; the other modes store to
      // global memory and lose 2-8 % to the longer live ranges, so they keep node order)
      double nb[2 * NPT][4];
      if (MODE == FM_PREX) {
#pragma unroll
        for (int r = 0; r < NPT; ++r) {
          nbrs(k0, r, nb[2 * r]);
          nbrs(k0 + 1, r, nb[2 * r + 1]);
        }
      }
#pragma unroll
      for (int r = 0; r < NPT; ++r) {
        if (MODE != FM_PREX) nbrs(k0, r, nb[2 * r]);
        node(k0, r, gk, xd[r], xc[r], u0[r], bcv[r], nb[2 * r]);
        if (MODE != FM_PREX) nbrs(k0 + 1, r, nb[2 * r + 1]);
        node(k0 + 1, r, gk + N2, xc[r], u0[r], u1[r], b0[r], nb[2 * r + 1]);
      }
      gk += 2 * N2;
    } else {
      step(k0, xd, xc, u0, bcv);
      if (two) step(k0 + 1, xc, u0, u1, b0);
    }
#pragma unroll
    for (int r = 0; r < NPT; ++r) {
      xd[r] = u0[r];
      xc[r] = u1[r];
      bcv[r] = b1[r];
    }
    if (!XF) {
      __syncthreads();  // every thread is done with planes k0-1 .. k0+1
      if (tid == 0) {
        if (k0 - 1 + S <= p_last) issue(k0 - 1 + S);
        if (k0 + S <= p_last) issue(k0 + S);
      }
      if (MODE == FM_PREX && xon) {  // SW: this trip's r1 planes are complete (barrier above)
        const double v0 = xload(k0), v1 = two ? xload(k0 + 1) : 0.0;
        xz(k0, v0);
        if (two) xz(k0 + 1, v1);
      }
    }
  }
  if (MODE == FM_PREX && XF) {  // the last trip's planes
    __syncthreads();
    const int kl = kb + (((ke - kb) - 1) & ~1);
    if (xon) {
      xz(kl, xload(kl));
      if (kl + 1 < ke) xz(kl + 1, xload(kl + 1));
    }
  }
  if (a.dot != DOT_NONE) {
    __shared__ double red[32];
    const double s = block_reduce_sum(acc, red);
    if (tid == 0) a.partial[(int64_t)mu * a.g.tiles + yt * zc + kc] = s;
  }
}

template <int MODE, int N, bool DC, bool SCW = false, bool SW = false>
static cudaError_t fine_launch_mnd(const FineArgs& a, int batch, cudaStream_t stream) {
  using G = FTM<MODE, N>;
  const int np = a.g.kz + (MODE == FM_PREX ? 3 : 2);  // FM_PREX: one recomputed plane
  const size_t smem = FSmem<N, MODE, DC, SW>::bytes(np, SCW ? 0 : a.op.Q);
  cudaError_t e0 = cudaSuccess;
  if (a.g.threads != G::THREADS || a.g.ty != G::TY || smem > 227 * 1024)
    e0 = cudaErrorInvalidValue;
  else
    e0 = smem_attr((const void*)fine_kernel<MODE, N, DC, SCW, SW>, smem);
  if (e0 != cudaSuccess) {
    fprintf(stderr, "[rbws] fine_kernel<%d,%d,%d,%d,%d> not launched: threads %d/%d ty %d/%d kz %d "
            "smem %zu: %s\n", MODE, N, (int)DC, (int)SCW, (int)SW, a.g.threads, G::THREADS, a.g.ty, G::TY,
            a.g.kz, smem, cudaGetErrorString(e0));
    return e0;
  }
  dim3 grd(1, a.g.ytiles, batch * a.g.zc);
  count_launch();
  fine_kernel<MODE, N, DC, SCW, SW><<<grd, G::THREADS, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  static const bool dbg = getenv("RBWS_DEBUG_LAUNCH") != nullptr;
  if (dbg || e != cudaSuccess)
    fprintf(stderr, "[rbws] fine_kernel<%d,%d,%d,%d> grid (1,%d,%d) block %d smem %zu: %s\n",
            MODE, N, (int)DC, (int)SCW, a.g.ytiles, batch * a.g.zc, G::THREADS, smem,
            cudaGetErrorString(e));
  return e;
}

template <int MODE, int N>
static cudaError_t fine_launch_mn(const FineArgs& a, int batch, cudaStream_t stream) {
  if (a.op.wface) return fine_launch_mnd<MODE, N, false, true>(a, batch, stream);
  if constexpr (MODE == FM_PRE || MODE == FM_PREX)
    if (a.sw) return fine_launch_mnd<MODE, N, false, false, true>(a, batch, stream);
  if constexpr (MODE == FM_PAPPLY)
    if (g_direct_papply.load(std::memory_order_relaxed) && N <= 128)
      return fine_launch_mnd<MODE, N, false, false, true>(a, batch, stream);
  if constexpr (MODE == FM_PRE || MODE == FM_PREX || MODE == FM_POSTP)
    if (a.dc) return fine_launch_mnd<MODE, N, true>(a, batch, stream);
  return fine_launch_mnd<MODE, N, false>(a, batch, stream);
}

template <int MODE>
static cudaError_t fine_launch_m(const FineArgs& a, int batch, cudaStream_t stream) {
  switch (a.op.n) {
    case 8: return fine_launch_mn<MODE, 8>(a, batch, stream);
    case 16: return fine_launch_mn<MODE, 16>(a, batch, stream);
    case 32: return fine_launch_mn<MODE, 32>(a, batch, stream);
    case 64: return fine_launch_mn<MODE, 64>(a, batch, stream);
    case 128: return fine_launch_mn<MODE, 128>(a, batch, stream);
    case 256: return fine_launch_mn<MODE, 256>(a, batch, stream);
    case 512: return fine_launch_mn<MODE, 512>(a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

static cudaError_t fine_launch(int mode, FineArgs& a, int batch, cudaStream_t stream) {
  if (a.op.Q < 1 || a.op.Q > kMaxTerms) return cudaErrorInvalidValue;
  if (a.zhi <= 0) { a.zlo = 0; a.zhi = a.op.n; }
  a.g = fine_geom(a.op.n, batch, a.zhi - a.zlo, fine_mode_threads(mode, a.op.n));
  switch (mode) {
    case FM_APPLY: return fine_launch_m<FM_APPLY>(a, batch, stream);
    case FM_RESID: return fine_launch_m<FM_RESID>(a, batch, stream);
    case FM_JACOBI: return fine_launch_m<FM_JACOBI>(a, batch, stream);
    case FM_PRE: return fine_launch_m<FM_PRE>(a, batch, stream);
    case FM_PREX: return fine_launch_m<FM_PREX>(a, batch, stream);
    case FM_CG: return fine_launch_m<FM_CG>(a, batch, stream);
    case FM_PAPPLY: return fine_launch_m<FM_PAPPLY>(a, batch, stream);
    case FM_POSTP: return fine_launch_m<FM_POSTP>(a, batch, stream);
    default: return cudaErrorInvalidValue;
  }
}

// Stored face weights of every instance (batch setup of the SCW kernels): for node
// (i, j, k) the weight of its +x, +y, +z face, with the same expression and summation
// order as the kernels' register refresh (fine_kernel::weights), so both paths agree
// bitwise.  Faces on the Dirichlet boundary planes (a coordinate 0) are included where a
// kernel reads them as the -x / -y / -z face of an interior node.
template <int Q>
__global__ void __launch_bounds__(256) fine_faces_kernel(Sep7 op, int n, double* __restrict__ wx,
                                                        double* __restrict__ wy,
                                                        double* __restrict__ wz) {
  const int n1 = n + 1;
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
  const int mu = blockIdx.z;
  const int64_t X = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= n3) return;
  const int i = X % n, j = (X / n) % n, k = (int)(X / n2);
  const double* th = op.theta + (size_t)mu * Q;
  double a0 = 0.0, a2 = 0.0, a4 = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double* F = op.face + (size_t)q * 3 * n;
    const double* NF = op.node + (size_t)q * 9 * n1;
    const double t = th[q];
    const double zx = NF[(0 * 3 + 2) * n1 + k], zy = NF[(1 * 3 + 2) * n1 + k];
    const double zz = (k < n) ? F[2 * n + k] : 0.0;
    const double tx = t * NF[(0 * 3 + 1) * n1 + j] * zx;
    const double tyv = t * NF[(1 * 3 + 0) * n1 + i] * zy;
    const double tz = t * NF[(2 * 3 + 0) * n1 + i] * NF[(2 * 3 + 1) * n1 + j];
    a0 = fma(F[0 * n + i], tx, a0);
    a2 = fma(F[1 * n + j], tyv, a2);
    a4 = fma(tz, zz, a4);
  }
  const int64_t o = (int64_t)mu * n3 + X;
  wx[o] = (j >= 1 && k >= 1) ? a0 : 0.0;
  wy[o] = (i >= 1 && k >= 1) ? a2 : 0.0;
  wz[o] = (i >= 1 && j >= 1) ? a4 : 0.0;
}

cudaError_t fine_faces(const Sep7& op, int batch, double* wface, int64_t wstride,
                       cudaStream_t stream) {
  const int n = op.n;
  const int64_t n3 = (int64_t)n * n * n;
  dim3 grd((unsigned)((n3 + 255) / 256), 1, batch);
  count_launch();
#define RBWS_FQ(QQ) \
  case QQ: fine_faces_kernel<QQ><<<grd, 256, 0, stream>>>(op, n, wface, wface + wstride, \
                                                          wface + 2 * wstride); break;
  switch (op.Q) {
    RBWS_FQ(1) RBWS_FQ(2) RBWS_FQ(3) RBWS_FQ(4) RBWS_FQ(5) RBWS_FQ(6) RBWS_FQ(7) RBWS_FQ(8)
    default: return cudaErrorInvalidValue;
  }
#undef RBWS_FQ
  return cudaGetLastError();
}

// 1/diag of the finest operator for every instance (batch setup); weights are
// recomputed only on planes whose z factors change (host-built flags)
template <int Q>
__global__ void __launch_bounds__(512) fine_dinv_kernel(Sep7 op, FineGeom g, const int* zsame,
                                                       double* __restrict__ dinv, int zlo,
                                                       int zhi) {
  const int n = op.n, n1 = n + 1;
  const int kc = blockIdx.z % g.zc, mu = blockIdx.z / g.zc;
  const int kz = g.kz;
  const int kb = max(1, zlo + kc * kz), ke = min(min(n, zhi), zlo + (kc + 1) * kz);
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
                      cudaStream_t stream, int zlo, int zhi) {
  if (zhi <= 0) { zlo = 0; zhi = op.n; }
  const FineGeom g = fine_geom(op.n, batch, zhi - zlo);
  dim3 grd(1, g.ytiles, batch * g.zc);
  count_launch();
#define RBWS_DQ(QQ) \
  case QQ: fine_dinv_kernel<QQ><<<grd, g.threads, 0, stream>>>(op, g, zsame, dinv, zlo, zhi); break;
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
  a.zlo = lc.zlo;
  a.zhi = lc.zhi;
  // few planes where the diagonal changes along z: cache w/diag instead of reading dinv.
  // Measured: at N <= 128 (two 256-thread CTAs per SM) the transformed-input kernels are
  // issue-bound and the saved 8 B/node buy nothing; at N = 512 (one CTA per SM) they do.
  const int force = g_force_dc.load(std::memory_order_relaxed);
  const bool few = op.fz && op.zchg >= 0 && op.zchg <= kMaxDiagChanges;
  a.dc = (few && (force < 0 ? op.n >= 256 : force == 1)) ? 1 : 0;
  a.sw = (few && !op.wface && g_force_sw.load(std::memory_order_relaxed) != 0) ? 1 : 0;
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

template <int N>
static size_t prex_smem(bool dc, bool sw, int np, int Q) {
  if (sw) return FSmem<N, FM_PREX, false, true>::bytes(np, Q);
  return dc ? FSmem<N, FM_PREX, true>::bytes(np, Q) : FSmem<N, FM_PREX, false>::bytes(np, Q);
}

bool fine_pre_scaled(const Sep7& op) {
  return base_args(op, DOT_NONE, nullptr, LaunchCtx{}, 0.0).sw != 0;
}

bool fine_pre_xz_ok(const Sep7& op, int batch, const LaunchCtx& lc) {
  const int n = op.n;
  if (lc.zhi > 0 && (lc.zlo != 0 || lc.zhi != n)) return false;  // z-ranges (slabs): no
  static const bool n128 = [] {  // A/B: RBWS_FUSED_N128=0 keeps the separate kernels
    const char* e = getenv("RBWS_FUSED_N128");
    return !(e && atoi(e) == 0);
  }();
  // N = 128: the r1 double buffer (16 KB) on top of the 4-slot ring cost the second CTA per
  // SM (configs[2]: pre + restriction 7.4 -> 10.4 ms per V-cycle); FM_PREX runs a 3-slot ring
  // there: 7.37 -> 7.27 ms, 792 -> 813 solves/s (A/B, two runs each)
  if (n == 128 && !n128) return false;
  // z-chunks must start on even planes (a chunk then recomputes the odd plane below it)
  const FineGeom g = fine_geom(n, batch, n, fine_mode_threads(FM_PREX, n));
  if (g.kz & 1) return false;
  // the z-factor table grows with the chunk's planes: at N = 512 with a short batch (long
  // chunks) it no longer fits next to the ring -> separate pre-smoothing + restriction
  const int Q = op.wface ? 0 : op.Q, np = g.kz + 3;
  const FineArgs ba = base_args(op, DOT_NONE, nullptr, lc, 0.0);
  const bool dc = ba.dc != 0, sw = ba.sw != 0;
  size_t smem = 0;
  switch (n) {
    case 8: smem = prex_smem<8>(dc, sw, np, Q); break;
    case 16: smem = prex_smem<16>(dc, sw, np, Q); break;
    case 32: smem = prex_smem<32>(dc, sw, np, Q); break;
    case 64: smem = prex_smem<64>(dc, sw, np, Q); break;
    case 128: smem = prex_smem<128>(dc, sw, np, Q); break;
    case 256: smem = prex_smem<256>(dc, sw, np, Q); break;
    case 512: smem = prex_smem<512>(dc, sw, np, Q); break;
    default: return false;
  }
  return smem <= 227 * 1024;
}

cudaError_t fine_pre_xz(const Sep7& op, int batch, const double* b, const double* dinv,
                        double* t, double omega, const LaunchCtx& lc) {
  if (!fine_pre_xz_ok(op, batch, lc)) return cudaErrorInvalidValue;
  FineArgs a = base_args(op, DOT_NONE, nullptr, lc, omega);
  a.h0 = b;
  a.h1 = dinv;
  a.out0 = t;
  return fine_launch(FM_PREX, a, batch, lc.stream);
}

cudaError_t fine_post_prolong(const Sep7& op, int batch, const double* b, const double* dinv,
                              const double* ec, double* y, double omega, double* partial,
                              const LaunchCtx& lc) {
  FineArgs a = base_args(op, partial ? DOT_BY : DOT_NONE, partial, lc, omega);
  a.h0 = b;
  a.h1 = dinv;
  a.ec = ec;
  a.out0 = y;
  return fine_launch(FM_POSTP, a, batch, lc.stream);
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
