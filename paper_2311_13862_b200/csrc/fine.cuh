// Finest-level kernels with TMA-engine plane staging (see fine.cu).
#pragma once

#include "stencil.cuh"

namespace rbws {

// override of the DC kernel choice (-1 auto: N >= 256; 0 never; 1 whenever applicable)
int fine_set_dc(int v);
// override of the scaled-weights pre-smoothing kernels (-1 / 1 auto, 0 never)
int fine_set_sw(int v);
// p-update kernel without the transformed ring (-1 / 1 on, 0 off)
int fine_set_direct(int v);
int fine_variant();  // current override (part of the cached PCG graph's key)

struct FineGeom {
  int threads;  // threads per CTA (rows-per-pass x n)
  int rpp;      // grid rows covered per pass of the CTA
  int npt;      // nodes per thread per plane
  int ty;       // rows per tile = rpp * npt
  int ytiles;   // tiles per plane
  int zc;       // z-chunks per instance
  int kz;       // planes per z-chunk
  int tiles;    // partial-sum slots per instance = ytiles * zc
};
// nz: planes per instance processed (0 = n; slabs pass their owned plane count)
FineGeom fine_geom(int n, int batch, int nz = 0, int threads = 0);
// threads per CTA of fine kernel mode `mode` on an n-cell grid (geometry of its dot partials)
int fine_mode_threads(int mode, int n);
// partial-sum slots per instance of the prolongation + post-smoothing kernel (the V-cycle's dot)
inline int fine_post_tiles(int n, int batch, int nz = 0) {
  return fine_geom(n, batch, nz, fine_mode_threads(6, n)).tiles;
}

// y = A x (y may be null), partial (may be null) = x . A x
cudaError_t fine_apply(const Sep7& op, int batch, const double* x, double* y, double* partial,
                       const LaunchCtx& lc);
// r = b - A x (r may be null: norm only), partial = |r|^2 (b_shared: b is one instance used
// by every instance)
cudaError_t fine_resid(const Sep7& op, int batch, const double* x, const double* b, double* r,
                       double* partial, const LaunchCtx& lc, bool b_shared = false);
// dinv = 1/diag(A(mu)) (batch setup); zsame: per-plane "z factors unchanged" flags
cudaError_t fine_dinv(const Sep7& op, int batch, const int* zsame, double* dinv,
                      cudaStream_t stream, int zlo = 0, int zhi = 0);
// y = x + omega (b - A x)/diag, partial (may be null) = b . y
cudaError_t fine_jacobi(const Sep7& op, int batch, const double* x, const double* b, double* y,
                        double omega, double* partial, const LaunchCtx& lc);
// r1 = b - A (omega dinv b)
cudaError_t fine_pre(const Sep7& op, int batch, const double* b, const double* dinv, double* r1,
                     double omega, const LaunchCtx& lc);
// pre-smoothing residual fused with the x and z passes of the restriction:
// t[K][j][I] (n/2 x n x n/2 per instance) = sum over fine planes 2K-1..2K+1 and columns
// 2I-1..2I+1 (weights 0.5 / 1 / 0.5) of r1 = b - A (omega dinv b) on fine row j; the y pass is
// restrict_y_launch.  Only when one CTA holds an instance's whole z-range (fine_pre_xz_ok).
bool fine_pre_xz_ok(const Sep7& op, int batch, const LaunchCtx& lc);
// true when fine_pre / fine_pre_xz run the scaled-weights kernels on this operator (no 1/diag
// stream: the measurement's byte counts)
bool fine_pre_scaled(const Sep7& op);
cudaError_t fine_pre_xz(const Sep7& op, int batch, const double* b, const double* dinv,
                        double* t, double omega, const LaunchCtx& lc);
// fused prolongation + post-smoothing of the nu=1 V-cycle:
// u = w dinv b + P ec (ec: coarse correction, n/2 cells), y = u + w (b - A u)/diag,
// partial (may be null) = b . y
cudaError_t fine_post_prolong(const Sep7& op, int batch, const double* b, const double* dinv,
                              const double* ec, double* y, double omega, double* partial,
                              const LaunchCtx& lc);
// stored face weights (+x, +y, +z face of every node) for the SCW kernels: wface holds three
// padded batch vectors at stride wstride doubles
cudaError_t fine_faces(const Sep7& op, int batch, double* wface, int64_t wstride,
                       cudaStream_t stream);
// planes with a new diagonal above which the stored-weight kernels are used
constexpr int kFineStoredWeightsMinChanges = 17;
// x += alpha p, r -= alpha A p, partial = |r|^2
cudaError_t fine_cg_update(const Sep7& op, int batch, const double* p, double* x, double* r,
                           const double* alpha, double* partial, const LaunchCtx& lc);
// The CG update fused with the next V-cycle's pre-smoothing residual and the x/z passes of its
// restriction (cgp.cu): x += alpha p, r -= alpha A p, partial = |r|^2 (the CG update kernel's
// slots), t = x/z-restricted r - A (omega D^-1 r) (the layout of fine_pre_xz).
bool fine_cgp_ok(const Sep7& op, int batch, const LaunchCtx& lc);
int fine_set_cgp(int v);    // 1 on where it applies, -1 / 0 off
int fine_cgp_variant();
// r_out != r_in: the tiles read each other's old rows as halos while they update
cudaError_t fine_cg_update_pre(const Sep7& op, int batch, const double* p, double* x,
                               const double* r_in, double* r_out, const double* alpha,
                               double* partial, double* t, double omega, const LaunchCtx& lc);
// p_new = s + beta p_old (beta null: p_new = s), partial = p_new . A p_new
cudaError_t fine_papply(const Sep7& op, int batch, const double* s, const double* p_old,
                        const double* beta, double* p_new, double* partial, const LaunchCtx& lc);

}  // namespace rbws

