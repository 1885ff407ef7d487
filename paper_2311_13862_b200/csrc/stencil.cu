// Batched stencil / transfer / vector kernels (sm_100a).
//
// Finest level: matrix-free separable 7-point operator.  One thread owns a
// grid column (i, j) of one parameter instance and marches in z: the
// Kronecker factors of the affine terms reduce to 5Q per-column constants
// held in registers, so each face weight costs Q FMAs and the z-neighbours
// of the input stay in registers.  Lateral neighbours come through L1.
// Coarse levels: per-instance symmetric 27-point stencils (14 stored
// coefficients per node) produced by the batched affine assembly st27_build.
#include "stencil.cuh"

namespace rbws {

// ========================================================================
// finest level: separable 7-point
// ========================================================================

Sep7Geom sep7_geom(int n, int batch) {
  Sep7Geom g;
  g.tx = n < 32 ? n : 32;
  g.ty = 256 / g.tx;
  if (g.ty > n) g.ty = n;
  int bxy = (n / g.tx) * (n / g.ty);
  g.zc = 1;
  while ((int64_t)bxy * batch * g.zc < 4 * 148 && g.zc * 8 <= n) g.zc *= 2;
  g.tiles = bxy * g.zc;
  return g;
}

template <int Q>
struct ColConst {
  double cxp[Q], cxm[Q], cyp[Q], cym[Q], cz[Q];
  const double* zx[Q];  // node factor along z of the x-part
  const double* zy[Q];  // node factor along z of the y-part
  const double* fz[Q];  // face factor along z of the z-part

  __device__ __forceinline__ void init(const Sep7& op, int mu, int i, int j) {
    const int n = op.n, n1 = n + 1;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double t = op.theta[mu * Q + q];
      const double* F = op.face + (size_t)q * 3 * n;
      const double* N = op.node + (size_t)q * 9 * n1;
      const double nxy = N[(0 * 3 + 1) * n1 + j];  // x-part, along y
      const double nyx = N[(1 * 3 + 0) * n1 + i];  // y-part, along x
      cxp[q] = t * F[0 * n + i] * nxy;
      cxm[q] = t * F[0 * n + i - 1] * nxy;
      cyp[q] = t * F[1 * n + j] * nyx;
      cym[q] = t * F[1 * n + j - 1] * nyx;
      cz[q] = t * N[(2 * 3 + 0) * n1 + i] * N[(2 * 3 + 1) * n1 + j];
      zx[q] = N + (0 * 3 + 2) * n1;
      zy[q] = N + (1 * 3 + 2) * n1;
      fz[q] = F + 2 * n;
    }
  }
  __device__ __forceinline__ double wz(int k) const {  // z-face between k, k+1
    double w = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) w = fma(cz[q], __ldg(fz[q] + k), w);
    return w;
  }
  __device__ __forceinline__ void wxy(int k, double& wxp, double& wxm, double& wyp,
                                      double& wym) const {
    wxp = wxm = wyp = wym = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double a = __ldg(zx[q] + k), b = __ldg(zy[q] + k);
      wxp = fma(cxp[q], a, wxp);
      wxm = fma(cxm[q], a, wxm);
      wyp = fma(cyp[q], b, wyp);
      wym = fma(cym[q], b, wym);
    }
  }
};

template <int Q, int MODE>
__global__ void __launch_bounds__(256) sep7_kernel(Sep7 op, int zc, int dot,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ b,
                                                   const double* __restrict__ dinv,
                                                   double* __restrict__ y,
                                                   double* __restrict__ partial,
                                                   const int* __restrict__ active,
                                                   double omega) {
  __shared__ double red[32];
  const int n = op.n;
  const int kc = blockIdx.z % zc, mu = blockIdx.z / zc;
  if (active && !active[mu]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const bool valid = (i >= 1) && (j >= 1);
  const int kz = n / zc;
  const int kb = max(1, kc * kz), ke = min(n, (kc + 1) * kz);
  const int64_t n2 = (int64_t)n * n;
  const int64_t base = (int64_t)mu * n2 * n;
  double acc = 0.0;
  if (valid) {
    ColConst<Q> cc;
    cc.init(op, mu, i, j);
    const int64_t col = base + i + (int64_t)n * j;
    auto ld = [&](int64_t idx) -> double {
      if (MODE == MODE_PRE) return omega * __ldg(dinv + idx) * __ldg(b + idx);
      if (MODE == MODE_DINV) return 0.0;
      return __ldg(x + idx);
    };
    double um = ld(col + (int64_t)(kb - 1) * n2);
    double uc = ld(col + (int64_t)kb * n2);
    double wzm = cc.wz(kb - 1);
    for (int k = kb; k < ke; ++k) {
      const int64_t idx = col + (int64_t)k * n2;
      const double up = ld(idx + n2);
      const double ue = ld(idx + 1), uw = ld(idx - 1), un = ld(idx + n), us = ld(idx - n);
      double wxp, wxm, wyp, wym;
      cc.wxy(k, wxp, wxm, wyp, wym);
      const double wzp = cc.wz(k);
      const double d = ((wxp + wxm) + (wyp + wym)) + (wzp + wzm);
      double out;
      if (MODE == MODE_DINV) {
        out = 1.0 / d;
      } else {
        double off = wxp * ue;
        off = fma(wxm, uw, off);
        off = fma(wyp, un, off);
        off = fma(wym, us, off);
        off = fma(wzp, up, off);
        off = fma(wzm, um, off);
        const double Au = fma(d, uc, -off);
        if (MODE == MODE_APPLY) {
          out = Au;
        } else if (MODE == MODE_RESID || MODE == MODE_PRE) {
          out = __ldg(b + idx) - Au;
        } else {  // MODE_JACOBI
          out = uc + omega * (__ldg(b + idx) - Au) / d;
        }
        if (dot == DOT_XAX) acc = fma(uc, Au, acc);
      }
      if (dot == DOT_YY) acc = fma(out, out, acc);
      else if (dot == DOT_BY) acc = fma(__ldg(b + idx), out, acc);
      if (y) y[idx] = out;
      um = uc;
      uc = up;
      wzm = wzp;
    }
  }
  if (dot != DOT_NONE) {
    const double s = block_reduce_sum(acc, red);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      const int tile = (blockIdx.y * gridDim.x + blockIdx.x) * zc + kc;
      const int tiles = gridDim.x * gridDim.y * zc;
      partial[(int64_t)mu * tiles + tile] = s;
    }
  }
}

template <int Q>
static cudaError_t sep7_launch_q(const Sep7& op, int batch, int mode, int dot, const double* x,
                                 const double* b, const double* dinv, double* y,
                                 double* partial, double omega, const LaunchCtx& lc) {
  Sep7Geom g = sep7_geom(op.n, batch);
  dim3 blk(g.tx, g.ty), grd(op.n / g.tx, op.n / g.ty, batch * g.zc);
  count_launch();
#define RBWS_SEP7_CASE(M)                                                             \
  case M:                                                                             \
    sep7_kernel<Q, M><<<grd, blk, 0, lc.stream>>>(op, g.zc, dot, x, b, dinv, y, partial, \
                                                 lc.active, omega);                   \
    break;
  switch (mode) {
    RBWS_SEP7_CASE(MODE_APPLY)
    RBWS_SEP7_CASE(MODE_RESID)
    RBWS_SEP7_CASE(MODE_JACOBI)
    RBWS_SEP7_CASE(MODE_PRE)
    RBWS_SEP7_CASE(MODE_DINV)
    default:
      return cudaErrorInvalidValue;
  }
#undef RBWS_SEP7_CASE
  return cudaGetLastError();
}

#define RBWS_Q_DISPATCH(Qv, CALL)        \
  switch (Qv) {                          \
    case 1: return CALL(1);              \
    case 2: return CALL(2);              \
    case 3: return CALL(3);              \
    case 4: return CALL(4);              \
    case 5: return CALL(5);              \
    case 6: return CALL(6);              \
    case 7: return CALL(7);              \
    case 8: return CALL(8);              \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t sep7_launch(const Sep7& op, int batch, int mode, int dot, const double* x,
                        const double* b, const double* dinv, double* y, double* partial,
                        double omega, const LaunchCtx& lc) {
#define CALL(QQ) sep7_launch_q<QQ>(op, batch, mode, dot, x, b, dinv, y, partial, omega, lc)
  RBWS_Q_DISPATCH(op.Q, CALL)
#undef CALL
}

// ========================================================================
// transfers (trilinear prolongation and its transpose)
// ========================================================================

__global__ void __launch_bounds__(256) restrict_kernel(int nf, const double* __restrict__ rf,
                                                       double* __restrict__ bc,
                                                       const int* __restrict__ active,
                                                       const double* __restrict__ dinv_c,
                                                       double* __restrict__ uc, double omega,
                                                       int64_t x0, int64_t x1) {
  const int nc = nf / 2;
  const int mu = blockIdx.y;
  if (active && !active[mu]) return;
  const int64_t nc3 = (int64_t)nc * nc * nc, nf3 = (int64_t)nf * nf * nf;
  const int64_t X = x0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // coarse node
  if (X >= x1) return;
  const int I = X % nc, J = (X / nc) % nc, K = X / ((int64_t)nc * nc);
  if (I == 0 || J == 0 || K == 0) return;
  const double* r = rf + (int64_t)mu * nf3;
  const int64_t nf2 = (int64_t)nf * nf;
  const int64_t c = 2 * I + (int64_t)nf * 2 * J + nf2 * 2 * K;
  double acc = 0.0;
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz) {
    double pz = 0.0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int64_t row = c + dz * nf2 + dy * (int64_t)nf;
      const double px = 0.5 * (__ldg(r + row - 1) + __ldg(r + row + 1)) + __ldg(r + row);
      pz += (dy == 0 ? 1.0 : 0.5) * px;
    }
    acc += (dz == 0 ? 1.0 : 0.5) * pz;
  }
  const int64_t o = (int64_t)mu * nc3 + X;
  bc[o] = acc;
  if (uc) uc[o] = omega * __ldg(dinv_c + o) * acc;  // pre-scaled rhs of the coarse pre-smoother
}

cudaError_t restrict_launch(int nf, int batch, const double* rf, double* bc, const LaunchCtx& lc,
                            const double* dinv_c, double* uc, double omega) {
  const int nc = nf / 2;
  const int64_t nc2 = (int64_t)nc * nc;
  // coarse planes [zlo, zhi) (slab path) or the whole level
  const int64_t x0 = lc.zhi > 0 ? lc.zlo * nc2 : 0, x1 = lc.zhi > 0 ? lc.zhi * nc2 : nc2 * nc;
  dim3 blk(256), grd((unsigned)((x1 - x0 + 255) / 256), batch);
  count_launch();
  restrict_kernel<<<grd, blk, 0, lc.stream>>>(nf, rf, bc, lc.active, dinv_c, uc, omega, x0, x1);
  return cudaGetLastError();
}

// y pass of the restriction whose x and z passes ran inside the pre-smoothing kernel
// (fine_pre_xz): bc(I,J,K) = 0.5 t(K,2J-1,I) + t(K,2J,I) + 0.5 t(K,2J+1,I), t = n/2 x n x n/2
// per instance; with dinv_c/uc also uc = omega dinv_c bc
// (two coarse nodes I, I+1 per thread, 16-byte loads and stores; the ghost column I = 0 gets
// explicit zeros)
__global__ void __launch_bounds__(256) restrict_y_kernel(int nf, const double* __restrict__ t,
                                                         double* __restrict__ bc,
                                                         const int* __restrict__ active,
                                                         const double* __restrict__ dinv_c,
                                                         double* __restrict__ uc, double omega) {
  const int nc = nf / 2, nh = nc / 2;
  const int mu = blockIdx.y;
  if (active && !active[mu]) return;
  const int64_t nc3 = (int64_t)nc * nc * nc;
  const int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pair of coarse nodes
  if (P >= nc3 / 2) return;
  const int I = 2 * (int)(P % nh), J = (int)((P / nh) % nc), K = (int)(P / ((int64_t)nh * nc));
  if (J == 0 || K == 0) return;
  const double* tk = t + (int64_t)mu * nc * nf * nc + (int64_t)K * nf * nc + I;
  const double2 a = __ldg(reinterpret_cast<const double2*>(tk + (int64_t)(2 * J - 1) * nc));
  const double2 c = __ldg(reinterpret_cast<const double2*>(tk + (int64_t)(2 * J) * nc));
  const double2 d = __ldg(reinterpret_cast<const double2*>(tk + (int64_t)(2 * J + 1) * nc));
  double2 acc;
  acc.x = 0.0; acc.x += 0.5 * a.x; acc.x += c.x; acc.x += 0.5 * d.x;
  acc.y = 0.0; acc.y += 0.5 * a.y; acc.y += c.y; acc.y += 0.5 * d.y;
  if (I == 0) acc.x = 0.0;
  const int64_t o = (int64_t)mu * nc3 + 2 * P;
  *reinterpret_cast<double2*>(bc + o) = acc;
  if (uc) {
    const double2 di = __ldg(reinterpret_cast<const double2*>(dinv_c + o));
    double2 u;
    u.x = omega * di.x * acc.x;
    u.y = omega * di.y * acc.y;
    if (I == 0) u.x = 0.0;
    *reinterpret_cast<double2*>(uc + o) = u;
  }
}

cudaError_t restrict_y_launch(int nf, int batch, const double* t, double* bc, const LaunchCtx& lc,
                              const double* dinv_c, double* uc, double omega) {
  const int64_t nc3 = (int64_t)(nf / 2) * (nf / 2) * (nf / 2);
  dim3 grd((unsigned)((nc3 / 2 + 255) / 256), batch);
  count_launch();
  restrict_y_kernel<<<grd, 256, 0, lc.stream>>>(nf, t, bc, lc.active, dinv_c, uc, omega);
  return cudaGetLastError();
}

// z-marching trilinear prolongation: one thread per fine column (i, j); the
// xy-interpolated coarse values of the two bracketing coarse planes are kept in
// registers, so each fine node costs one coarse gather per two fine planes.
// (a thread owns the fine column pair (2 ip, 2 ip + 1) of row j: both columns interpolate from
// the same coarse entries, 16-byte loads / stores; the ghost column i = 0 receives P e = 0)
__global__ void __launch_bounds__(512) prolong_kernel(int nf, int mode, int ty, int zc,
                                                      const double* __restrict__ ec,
                                                      double* __restrict__ u,
                                                      const double* __restrict__ b,
                                                      const double* __restrict__ dinv,
                                                      double omega,
                                                      const int* __restrict__ active, int zlo,
                                                      int zhi) {
  const int nc = nf / 2;
  const int mu = blockIdx.z / zc, kc = blockIdx.z % zc;
  if (active && !active[mu]) return;
  const int ip = threadIdx.x % nc;
  const int j = blockIdx.y * ty + threadIdx.x / nc;
  if (j == 0) return;
  const int64_t nf2 = (int64_t)nf * nf, nc2 = (int64_t)nc * nc;
  const double* e = ec + (int64_t)mu * nc2 * nc + ip + (int64_t)nc * (j >> 1);
  const bool oj = j & 1;
  // coarse plane K interpolated to (2 ip, j) and (2 ip + 1, j)
  auto vxy = [&](int K, double& ve, double& vo) {
    const double* q = e + nc2 * K;
    const double q0 = __ldg(q), q1 = __ldg(q + 1);
    const double r0e = q0, r0o = 0.5 * (q0 + q1);
    if (!oj) {
      ve = r0e;
      vo = r0o;
      return;
    }
    const double p0 = __ldg(q + nc), p1 = __ldg(q + nc + 1);
    ve = 0.5 * (r0e + p0);
    vo = 0.5 * (r0o + 0.5 * (p0 + p1));
  };
  const int kz = (zhi - zlo + zc - 1) / zc;
  const int kb = max(1, zlo + kc * kz), ke = min(min(nf, zhi), zlo + (kc + 1) * kz);
  if (kb >= ke) return;
  int Kc = kb >> 1;
  double e0, o0, e1, o1;
  vxy(Kc, e0, o0);
  vxy(Kc + 1, e1, o1);
  const int64_t col = (int64_t)mu * nf2 * nf + 2 * ip + (int64_t)nf * j;
  for (int k = kb; k < ke; ++k) {
    const int K = k >> 1;
    if (K != Kc) {  // advance one coarse plane
      e0 = e1;
      o0 = o1;
      vxy(K + 1, e1, o1);
      Kc = K;
    }
    const double pe = (k & 1) ? 0.5 * (e0 + e1) : e0;
    const double po = (k & 1) ? 0.5 * (o0 + o1) : o0;
    const int64_t idx = col + (int64_t)k * nf2;
    double2* up = reinterpret_cast<double2*>(u + idx);
    double2 v;
    if (mode == 0) {
      v = *up;
      v.x += pe;
      v.y += po;
    } else if (mode == 2) {  // b holds the pre-scaled rhs w D^-1 b
      const double2 bv = __ldg(reinterpret_cast<const double2*>(b + idx));
      v.x = bv.x + pe;
      v.y = bv.y + po;
    } else {
      const double2 bv = __ldg(reinterpret_cast<const double2*>(b + idx));
      const double2 dv = __ldg(reinterpret_cast<const double2*>(dinv + idx));
      v.x = fma(omega * dv.x, bv.x, pe);
      v.y = fma(omega * dv.y, bv.y, po);
    }
    *up = v;
  }
}

cudaError_t prolong_launch(int nf, int batch, int mode, const double* ec, double* u,
                           const double* b, const double* dinv, double omega,
                           const LaunchCtx& lc) {
  const int nc = nf / 2;
  int ty = 256 / nc;
  if (ty < 1) ty = 1;
  if (ty > nf) ty = nf;
  while (nf % ty) --ty;
  const int threads = ty * nc;
  const int zlo = lc.zhi > 0 ? lc.zlo : 0, zhi = lc.zhi > 0 ? lc.zhi : nf;
  int zc = 1;
  while ((int64_t)(nf / ty) * batch * zc < 4 * 148 && (zhi - zlo) / (zc * 2) >= 4) zc *= 2;
  dim3 grd(1, nf / ty, batch * zc);
  count_launch();
  prolong_kernel<<<grd, threads, 0, lc.stream>>>(nf, mode, ty, zc, ec, u, b, dinv, omega,
                                                 lc.active, zlo, zhi);
  return cudaGetLastError();
}


// ========================================================================
// coarsest level: dense Cholesky per instance
// ========================================================================

// one warp per instance: forward then backward substitution
__global__ void coarse_solve_kernel(int n0, int batch, const double* __restrict__ Lall,
                                    const double* __restrict__ b, double* __restrict__ x,
                                    const int* __restrict__ active) {
  extern __shared__ double sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mu = blockIdx.x * (blockDim.x >> 5) + warp;
  if (mu >= batch) return;
  if (active && !active[mu]) return;
  const int m1 = n0 - 1, m = m1 * m1 * m1;
  double* y = sh + warp * m;
  const int64_t n3 = (int64_t)n0 * n0 * n0;
  const double* L = Lall + (int64_t)mu * m * m;
  auto pad = [&](int r) -> int64_t {
    const int i = r % m1 + 1, j = (r / m1) % m1 + 1, k = r / (m1 * m1) + 1;
    return (int64_t)mu * n3 + i + (int64_t)n0 * (j + (int64_t)n0 * k);
  };
  for (int r = lane; r < m; r += 32) y[r] = b[pad(r)];
  __syncwarp();
  for (int r = 0; r < m; ++r) {  // L y = b
    double s = 0.0;
    for (int c = lane; c < r; c += 32) s = fma(L[r * m + c], y[c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = (y[r] - s) / L[r * m + r];
    __syncwarp();
  }
  for (int r = m - 1; r >= 0; --r) {  // L^T x = y
    double s = 0.0;
    for (int c = r + 1 + lane; c < m; c += 32) s = fma(L[c * m + r], y[c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = (y[r] - s) / L[r * m + r];
    __syncwarp();
  }
  for (int r = lane; r < m; r += 32) x[pad(r)] = y[r];
}

cudaError_t coarse_solve(int n0, int batch, const double* L, const double* b, double* x,
                         const LaunchCtx& lc) {
  const int m1 = n0 - 1, m = m1 * m1 * m1;
  const int wpb = 4;
  const size_t smem = (size_t)wpb * m * sizeof(double);
  count_launch();
  coarse_solve_kernel<<<(batch + wpb - 1) / wpb, 32 * wpb, smem, lc.stream>>>(n0, batch, L, b, x,
                                                                           lc.active);
  return cudaGetLastError();
}

// ========================================================================
// vector ops on padded batch vectors
// ========================================================================

__global__ void __launch_bounds__(256) scale_dinv_kernel(int64_t n3, double omega,
                                                         const double* __restrict__ dinv,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ u) {
  const int64_t base = (int64_t)blockIdx.y * n3;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n3;
       idx += (int64_t)gridDim.x * blockDim.x)
    u[base + idx] = omega * __ldg(dinv + base + idx) * __ldg(b + base + idx);
}

cudaError_t vec_scale_dinv(int n, int batch, double omega, const double* dinv, const double* b,
                           double* u, cudaStream_t stream) {
  const int64_t n3 = (int64_t)n * n * n;
  dim3 blk(256), grd((unsigned)((n3 + 1023) / 1024), batch);
  count_launch();
  scale_dinv_kernel<<<grd, blk, 0, stream>>>(n3, omega, dinv, b, u);
  return cudaGetLastError();
}

int vec_tiles(int n) {
  const int64_t n3 = (int64_t)n * n * n;
  int64_t t = (n3 + 2047) / 2048;  // 256 threads x 8 elements
  return (int)t;
}

__global__ void __launch_bounds__(256) dot_kernel(int64_t n3, const double* __restrict__ x,
                                                  int64_t xs, const double* __restrict__ y,
                                                  int64_t ys, double* __restrict__ partial,
                                                  const int* __restrict__ active) {
  __shared__ double red[32];
  const int mu = blockIdx.y;
  if (active && !active[mu]) return;
  const double* a = x + mu * xs;
  const double* b = y + mu * ys;
  double acc = 0.0;
  const int64_t start = (int64_t)blockIdx.x * 2048;
  for (int t = 0; t < 8; ++t) {
    const int64_t idx = start + t * 256 + threadIdx.x;
    if (idx < n3) acc = fma(__ldg(a + idx), __ldg(b + idx), acc);
  }
  const double s = block_reduce_sum(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)mu * gridDim.x + blockIdx.x] = s;
}

cudaError_t vec_dot_range(int64_t count, const double* x, const double* y, double* partial,
                          cudaStream_t stream) {
  dim3 blk(256), grd((unsigned)((count + 2047) / 2048), 1);
  count_launch();
  dot_kernel<<<grd, blk, 0, stream>>>(count, x, 0, y, 0, partial, nullptr);
  return cudaGetLastError();
}

cudaError_t vec_dot(int n, int batch, const double* x, int64_t x_stride, const double* y,
                    int64_t y_stride, double* partial, const LaunchCtx& lc) {
  const int64_t n3 = (int64_t)n * n * n;
  dim3 blk(256), grd(vec_tiles(n), batch);
  count_launch();
  dot_kernel<<<grd, blk, 0, lc.stream>>>(n3, x, x_stride, y, y_stride, partial, lc.active);
  return cudaGetLastError();
}

}  // namespace rbws
