/* rbws_b200.h — C ABI of the B200-native RBWS hot path.
 *
 * The reference (rbws, Python) binds its compiled hot loops through the
 * Cython module rbws._smoothers (csr_gauss_seidel / csr_jacobi,
 * reference _smoothers.pyx:14-45) and otherwise runs scipy.sparse / numpy.
 * This library replaces the whole data-parallel path those calls sit on —
 * operator application, smoothing sweeps, grid transfers, V-cycle, PCG and
 * the L1ROC online/offline kernels — batched over parameter instances.
 *
 * Conventions
 *  - All functions return 0 on success, non-zero on error;
 *    rbws_last_error() describes the last failure of the calling thread.
 *  - Array arguments marked (dev) are device pointers, (host) host pointers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - Grid vectors use the padded batch layout: instance `mu` of a level with
 *    n cells occupies doubles [mu*n^3, (mu+1)*n^3) indexed i + n*(j + n*k);
 *    interior (free) DoFs are i,j,k in [1, n-1], all other entries are 0.
 *    A buffer for `count` instances holds count*n^3 + 2*n^2 doubles (the
 *    trailing ghost region absorbs diagonal stencil reads of the last instance).
 *    Interior ordering inside the padded block equals the reference's free-DoF
 *    ordering (lexicographic, x fastest; reference grid.py:1-5,
 *    problems.py:63-75).
 *  - Separable operator tables of an n-cell finest grid with Q affine terms:
 *      face[(q*3+d)*n + i]           d-face factor between nodes i and i+1
 *      node[((q*3+d)*3+a)*(n+1)+j]   factor along axis a != d at node j
 *    The weight of the d-face between X and X+e_d is
 *      sum_q theta_q(mu) * face[q][d][X_d] * prod_{a != d} node[q][d][a][X_a].
 */
#ifndef RBWS_B200_H
#define RBWS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rbws_hierarchy rbws_hierarchy;
typedef struct rbws_batch rbws_batch;

/* Library version (major*10000 + minor*100 + patch). */
int rbws_version(void);
/* Last error message of the calling thread ("" if none). */
const char* rbws_last_error(void);
/* Kernel launches issued by this library so far (process-wide counter). */
int64_t rbws_launch_count(void);
/* Copy `bytes` of device data to host memory through mapped pinned staging (a
 * kernel store, not a copy-engine DMA), then synchronise `stream`.  Control-data
 * readbacks (the reference's `.item()` / numpy conversions of small arrays)
 * use it so they never queue behind a bulk solution download on another stream. */
int rbws_fetch(void* dst_host, const void* src_device, int64_t bytes, void* stream);

/* ---- hierarchy: mu-independent part of ParametricProblem -------------------
 * Replaces ParametricProblem.__init__ hierarchy/coarsening
 * (reference grid.py:203-236) and build_hierarchy (grid.py:163-170): nested
 * grids m0*2^i cells, trilinear prolongation, termwise Galerkin coarsening
 * (carried out on the 1D Kronecker factors of every affine term).
 * face/node: (host) separable tables of the finest grid (see above). */
int rbws_hierarchy_create(rbws_hierarchy** out, int n, int m0, int nterms,
                          const double* face, const double* node);
/* Assembled (FEM) problems — the reference's own ParametricProblem path: per-term
 * stiffness assembled on the finest grid, restricted to free DoFs and Galerkin-coarsened
 * term by term (grid.py:203-236); operator(mu, level) = sum_q theta_q A_q^level
 * (grid.py:246-255).  coef: (host) levels 0..L-1 concatenated, level l =
 * [nterms][14][n_l^3] symmetric 27-point coefficients in the padded layout (index 0 the
 * diagonal, 1..13 the lexicographically positive offsets (dx,dy,dz): dz=1 rows
 * 1 + 3(dy+1) + (dx+1), then (dx,1,0) at 11+dx, then (1,0,0) at 13), zero on ghosts.
 * Every level runs the stored-coefficient kernels; batches, V-cycles and MGCG use the
 * same entry points as separable problems (the rhs must be per instance). */
int rbws_hierarchy_create_stored(rbws_hierarchy** out, int n, int m0, int nterms,
                                 const double* coef);
int rbws_hierarchy_is_stored(const rbws_hierarchy* h);
/* y = A_q^level x for `count` padded vectors (one affine term, mu-independent): the
 * per-term products of the L1ROC projection (rb.py:200-201) on stored problems. */
int rbws_hierarchy_term_apply(const rbws_hierarchy* h, int level, int term, int count,
                              const double* x, double* y, void* stream);
int rbws_hierarchy_destroy(rbws_hierarchy* h);
int rbws_hierarchy_levels(const rbws_hierarchy* h);
int rbws_hierarchy_cells(const rbws_hierarchy* h, int level);
/* (host) copy of the 1D factors of `level`: Q*3*3*2*(cells+1) doubles */
int rbws_hierarchy_factors(const rbws_hierarchy* h, int level, double* out, int64_t capacity);

/* Host-only variant (no device needed): the 1D factors of `level` computed
 * from the separable tables, same layout as rbws_hierarchy_factors. */
int rbws_kron_factors(int n, int m0, int nterms, const double* face, const double* node,
                      int level, double* out, int64_t capacity);

/* ---- batch: mg_context_for for a batch of parameters -----------------------
 * Replaces mg_context_for / _finish_context (multigrid.py:154-202): per-mu
 * operators on every level, Jacobi diagonals, Cholesky of the coarsest level.
 * nu: sweeps per side (>= 1), omega: Jacobi damping (reference 0.7,
 * multigrid.py:27). */
int rbws_batch_create(rbws_batch** out, rbws_hierarchy* h, int capacity, int nu, double omega);
int rbws_batch_destroy(rbws_batch* b);
/* theta: (dev) [count][Q] affine weights theta_q(mu). Returns the number of
 * instances whose coarsest operator failed to factor in *n_bad (host). */
int rbws_batch_setup(rbws_batch* b, const double* theta, int count, int* n_bad, void* stream);

/* PCG iterations after the first run as one CUDA graph with a device-side WHILE
 * condition (no host synchronisation between iterations; cached per solve shape).
 * Default on (environment RBWS_GRAPH=0 turns it off); not used while the event
 * profiler or a streaming download is active. */
int rbws_batch_set_graph(rbws_batch* b, int enable);
/* Process-wide kernel-variant override for tests and A/B runs (no reference counterpart).
 * which 0 = "DC" finest pre/post-smoothing kernels (w/diag cached in shared memory, 1/diag
 * rows staged only on planes where the diagonal changes): value -1 auto (N >= 256),
 * 0 never, 1 whenever the diagonal changes on few planes (any N).
 * which 1 = "SW" scaled-weights pre-smoothing kernels: -1 / 1 auto (whenever the diagonal
 * changes on few planes and the face weights are not stored), 0 never (the transformed-ring
 * kernels that stage u = omega D^-1 b).
 * which 2 = fused coarse tail (every level with at most 16 cells per axis and the coarsest
 * solve in one kernel per instance, vectors in shared memory; bitwise the per-level kernels):
 * 1 on where it applies, -1 / 0 the per-level kernels (default: measured neutral on the
 * headline).
 * which 3 = p-update kernel that forms the neighbours' p = s + beta p_old where they are read
 * (no transformed ring, three CTAs per SM; bitwise the transformed-ring kernel): 1 on
 * (N <= 128, weights not stored), -1 / 0 the transformed-ring kernel (default: measured
 * slower).
 * which 4 = CG update fused with the next V-cycle's pre-smoothing residual and the x/z passes
 * of its restriction (cgp.cu; 64^3 grids, whole instances per CTA, Jacobi nu = 1): -1 / 1 on
 * where it applies, 0 the separate kernels. */
int rbws_set_kernel_variant(int which, int value);
/* Smoother of the V-cycle: 0 damped Jacobi (the reference default for isotropic problems,
 * multigrid.py:183-188), 1 Gauss-Seidel (smoother="gs": nu forward lexicographic sweeps
 * before and nu backward sweeps after the coarse correction, multigrid.py:132-152, sweep
 * _smoothers.pyx:14-28).  Call before rbws_batch_setup; Gauss-Seidel allocates stored
 * fine face weights and coarse coefficients (the hyperplane-ordered sweeps read them). */
int rbws_batch_set_smoother(rbws_batch* b, int kind);
/* In-place Gauss-Seidel sweep(s) on `level` for every instance of a batch set up with
 * smoother 1: kind 1 forward, 2 backward, 3 symmetric (forward then backward; the MSRB
 * FINE_SMOOTH, reference msrb.py:20, kernels.py:93-95).  x, rhs: (dev) padded. */
int rbws_smooth(rbws_batch* b, int level, int kind, double* x, const double* rhs, void* stream);
/* 1 if the finest-level kernels of this batch read stored face weights (coefficients
 * whose z factors change on most planes; +24 B per node per stencil sweep), else 0 */
int rbws_batch_stored_weights(const rbws_batch* b);
/* 1 if the last V-cycle ran the finest pre-smoothing residual fused with the x/z passes of
 * the restriction (r1 = b - A(w D^-1 b) never written; the measurement's byte counts) */
int rbws_batch_fused_restrict(const rbws_batch* b);
/* 1 if the last V-cycle's finest pre-smoothing residual ran the scaled-weights kernels
 * (face weights pre-multiplied by the neighbours' omega/diag in registers, stencil taken on
 * the raw b: the 1/diag vector is not streamed; piecewise-constant coefficients), else 0 */
int rbws_batch_pre_scaled(const rbws_batch* b);
/* 1 if the last solve's CG update (x += alpha p, r -= alpha A p, krylov.py:89-92) also computed
 * the next V-cycle's pre-smoothing residual and the x/z passes of its restriction in the same
 * pass (r never re-read: 42 instead of 40 + 10 B per node; the measurement's byte counts) */
int rbws_batch_cg_fused(const rbws_batch* b);

/* y = A^level(mu) x for every instance (ParametricProblem.operator(mu, level) @ x,
 * grid.py:246-255).  x, y: (dev) padded vectors of that level. */
int rbws_apply(rbws_batch* b, int level, const double* x, double* y, void* stream);
/* One damped-Jacobi sweep y = x + omega (rhs - A x)/diag on `level`
 * (replaces _smoothers.pyx:31 csr_jacobi via Smoother._jacobi, kernels.py:98-115). */
int rbws_jacobi_sweep(rbws_batch* b, int level, const double* x, const double* rhs, double* y,
                      void* stream);
/* bc = P^T rf (multigrid.py:220 `P.T @ r`); nf = fine cells. (dev) */
int rbws_restrict(int nf, int count, const double* rf, double* bc, void* stream);
/* u += P ec (multigrid.py:221 `u + P @ e`). (dev) */
int rbws_prolong_add(int nf, int count, const double* ec, double* u, void* stream);
/* One V-cycle from zero on the finest level (mg_vcycle, multigrid.py:205-222). (dev) */
int rbws_vcycle(rbws_batch* b, const double* rhs, double* out, void* stream);

/* Batched MGCG (pcg_solve with the V-cycle preconditioner, krylov.py:42-109,
 * multigrid.py:225-232).
 * f: (dev) rhs, per instance stride f_stride doubles (0 = shared by all).
 * x: (dev) in: initial guesses, out: solutions.
 * iters [count], hist [count][l_max+1] (NaN padded), true_res [count],
 * status [count]: (host) outputs; status bit0 = breakdown (non-SPD),
 * bit1 = not converged, bit2 = ||f|| = 0 (absolute norms). */
int rbws_mgcg_solve(rbws_batch* b, const double* f, int64_t f_stride, double* x, double delta,
                    int l_max, int* iters, double* hist, double* true_res, int* status,
                    void* stream);

/* Batched PCG with the iteration-indexed multispace reduced-basis preconditioner
 * (msrbcg_solve, msrb.py:152-170, as called by rbi_pcg_solve, warmstart.py:103-104): from the
 * loaded x (the POD Galerkin initial guess), iteration k is preconditioned by one symmetric
 * Gauss-Seidel sweep from zero plus the Galerkin correction of its residual in basis
 * min(k, nbases - 1) (MsrbPreconditioner.__call__, msrb.py:77-85).  The batch must be set up
 * with smoother = 1.  Host arrays of nbases entries: W[k] (dev) N[k] <= 64 padded basis
 * vectors at stride Wstride[k]; chol[k] (dev) [count][N[k]][N[k]] lower Cholesky factors of
 * W_k^T A(mu) W_k (cho_factor, msrb.py:72).  Outputs as rbws_mgcg_solve. */
int rbws_msrbcg_solve(rbws_batch* b, const double* f, int64_t f_stride, double* x, double delta,
                      int l_max, int nbases, const double* const* W, const int64_t* Wstride,
                      const int* N, const double* const* chol, int* iters, double* hist,
                      double* true_res, int* status, void* stream);

/* rbws_mgcg_solve that also streams the solutions to host memory: instance m's
 * padded solution (n^3 doubles) is copied to x_host + m*host_stride (pinned host,
 * host_stride >= n^3) on copy_stream as soon as m stops iterating (converged,
 * breakdown, or l_max), overlapping the downloads with the iterations of the
 * instances still running.  All copies are enqueued on copy_stream when the call
 * returns (record an event there to know when x_host is complete). */
int rbws_mgcg_solve_to_host(rbws_batch* b, const double* f, int64_t f_stride, double* x,
                            double delta, int l_max, int* iters, double* hist, double* true_res,
                            int* status, void* stream, double* x_host, int64_t host_stride,
                            void* copy_stream);

/* One smoothing-level kernel on `level` (>= 1): mode 0 y = A x, 1 y = rhs - A x,
 * 2 y = x + omega (rhs - A x)/diag, 3 y = rhs - A (omega dinv rhs) (the nu=1
 * pre-smoothing residual, multigrid.py:218-219).  (dev) padded vectors. */
int rbws_level_kernel(rbws_batch* b, int level, int mode, const double* x, const double* rhs,
                      double* y, void* stream);
/* Copy of the per-instance Jacobi inverse diagonals 1/diag(A^level(mu)) of a
 * set-up batch into `out` (dev, padded layout of that level). */
int rbws_batch_dinv(rbws_batch* b, int level, double* out, void* stream);

/* Optional per-kernel-class timing with CUDA events on the launch stream
 * (enable resets the counters).  Classes (9): fine apply+dot, fine CG update,
 * fine pre-smooth+residual, fine restriction, fine prolongation, fine
 * post-smooth, p-update, all coarse levels, per-instance scalar kernels.
 * ms/calls: (host) arrays of nclass entries. */
int rbws_batch_profile(rbws_batch* b, int enable);
int rbws_batch_profile_read(rbws_batch* b, double* ms, int64_t* calls, int64_t* units,
                            int nclass);

/* ---- L1ROC reduced model (reference rb.py) -------------------------------- */
/* Term-wise sampled projections Bq[q][m][c] = (A_q W)[rows[m], c]
 * (the affine pieces of rb.py:200-201 `A[rows,:] @ basis`).
 * W: (dev) N padded finest-level vectors (stride Wstride doubles);
 * rows: (dev) padded node indices [M]; Bq: (dev) [Q][M][N]. */
int rbws_l1roc_project(rbws_hierarchy* h, const double* W, int64_t Wstride, int N,
                       const int64_t* rows, int M, double* Bq, void* stream);
/* Batched online stage (rb.py:182-205, 129-131): B(mu) = sum_q theta_q Bq,
 * least squares min ||B a - b_s||, snapshot coordinates c = T^{-1} a and
 * indicator ||c||_1.  theta (dev) [count][Q]; bs (dev) [M] per instance with
 * stride bs_stride (0 = shared); T (dev) [N][N] row-major upper triangular
 * (may be NULL: no indicator).  Outputs (dev): a [count][N], c [count][N],
 * ind [count], status [count] (1 = rank deficient). */
int rbws_l1roc_online(int count, int Q, int M, int N, const double* theta, const double* Bq,
                      const double* bs, int64_t bs_stride, const double* T, double* a,
                      double* c, double* ind, int* status, void* stream);
/* out[m][a] = W[a] . v[m] for m < count, a < N: the basis projections W^T v of the
 * multispace preconditioner's Galerkin correction and the POD initial guess (reference
 * msrb.py:53-85, rb.py:71-83; `b @ W.T`).  W: (dev) N vectors of n3 doubles at stride
 * Wstride, v: (dev) count vectors at stride vstride, out: (dev) [count][N].  Deterministic
 * (fixed-order partial sums). */
int rbws_basis_dot(int64_t n3, int count, const double* W, int64_t Wstride, int N,
                   const double* v, int64_t vstride, double* out, void* stream);
/* x[mu] = W a[mu] (rb.py:205 `model.basis @ a`), (dev) padded output. */
int rbws_expand(int n, int count, const double* W, int64_t Wstride, int N, const double* a,
                double* x, void* stream);
/* DEIM residual step (rb.py:113-126): rho = v - W c, then the first index of
 * max |rho| over interior nodes not flagged in `excluded` (dev uint8, padded
 * layout, may be NULL), written with the pivot rho[idx] and max|v| to
 * out_idx (dev int64) / out_vals (dev double[2]); column = rho / pivot is
 * written to `col` (dev padded). */
int rbws_deim_step(int n, const double* W, int64_t Wstride, int N, const double* c,
                   const double* v, const uint8_t* excluded, double* col, int64_t* out_idx,
                   double* out_vals, void* stream);
/* The same DEIM step on full-node vectors ((side)^3 nodes per instance, fem_fn layout of
 * problems with free boundary nodes, example-2): every node is admissible (Dirichlet nodes
 * hold zeros; the free x = 1 face keeps its edge nodes, problems.py:63-75). */
int rbws_deim_step_fn(int side, const double* W, int64_t Wstride, int N, const double* c,
                      const double* v, const uint8_t* excluded, double* col, int64_t* out_idx,
                      double* out_vals, void* stream);
/* Small dense solve A x = b (partial pivoting) on the device, A (dev) [m][m]
 * row-major, b/x (dev) [m] (np.linalg.solve in rb.py:113). */
int rbws_dense_solve(int m, const double* A, const double* b, double* x, int* status,
                     void* stream);

/* ---- slab-decomposed single instance (BASELINE configs[4]) ----------------
 * One large instance of pcg_solve + mg_vcycle (krylov.py:42-109,
 * multigrid.py:205-232) with every level cut into `nslabs` slabs of whole
 * z-planes; slab r owns planes [r n_l/nslabs, (r+1) n_l/nslabs) of level l.
 * Coarse levels with fewer than 8 planes per slab are replicated.  Slabs in
 * one process exchange halo planes with device copies; across processes (one
 * per GPU) with NCCL send/recv, and dot-product partials are all-gathered, so
 * every slab computes bitwise identical PCG scalars.
 *   nccl_id: (host) 128 bytes from rbws_comm_unique_id on process 0, shared
 *            by every process.  NULL: all slabs live in this process and
 *            exchange by device copies; with nprocs == 1 and an id, the slabs
 *            of this process exchange through NCCL send/recv to itself
 *            (loopback: the multi-process code path on one GPU);
 *   nprocs/proc_rank: processes and this process's rank (slabs are assigned
 *            in process order: first = proc_rank * nlocal). */
typedef struct rbws_slab rbws_slab;
int rbws_comm_unique_id(uint8_t* out128);
int rbws_slab_create(rbws_slab** out, rbws_hierarchy* h, int nslabs, int nlocal,
                     const uint8_t* nccl_id, int nprocs, int proc_rank, double omega);
int rbws_slab_destroy(rbws_slab* s);
/* distributed levels start at *first_dist_level; owned planes of local slab i */
int rbws_slab_info(const rbws_slab* s, int* first_dist_level, int local, int* k0, int* k1);
/* mg_context_for for one parameter: theta (dev or host) [Q] */
int rbws_slab_setup(rbws_slab* s, const double* theta, int* n_bad, void* stream);
/* which: 0 = solution x, 1 = rhs f.  Copies the owned planes that fall in global
 * planes [p0, p0 + planes) from / to `buf` (device or host pointer holding those
 * planes of one padded instance, n^2 doubles per plane). */
int rbws_slab_load(rbws_slab* s, int which, const double* buf, int64_t p0, int planes,
                   void* stream);
int rbws_slab_store(rbws_slab* s, int which, double* buf, int64_t p0, int planes, void* stream);
/* x = P ec on the owned planes: a warm start prolonged from a full coarse
 * solution ec (dev, n/2 cells, one padded instance) */
int rbws_slab_prolong_x(rbws_slab* s, const double* ec, void* stream);
/* PCG to delta from the loaded x; outputs (host) as rbws_mgcg_solve for one instance */
int rbws_slab_solve(rbws_slab* s, double delta, int l_max, int* iters, double* hist,
                    double* true_res, int* status, void* stream);

/* ---- full-node ("FN") layout: assembled problems with free boundary nodes ----
 * (reference example-2, problems.py:135-152: zero-flux face x = 1).  One instance
 * = all (c+1)^3 nodes of a level (x fastest), Dirichlet nodes held at zero.  coef /
 * coefA: 27-point full-node coefficients [27][(c+1)^3], A[X, X+o] with
 * o = (dx+1) + 3(dy+1) + 9(dz+1); per term (coef, batch-shared) or per instance
 * (coefA).  All pointers device, streams cudaStream_t. */
/* coefA[i] = sum_q theta[i][q] coef[q] — ParametricProblem.operator, grid.py:246-255 */
int rbws_fn_combine(int count, int nterms, int c, const double* theta, const double* coef,
                    double* coefA, void* stream);
/* mode 0: y = A x; mode 1: y = b - A x — A @ x in multigrid.py:218, kernels.py:98-115 */
int rbws_fn_apply(int count, int c, const double* coefA, const double* x, const double* b,
                  double* y, int mode, void* stream);
/* the same from the batch-shared per-term coef [Q][27][(c+1)^3] and theta [count][Q]
 * (no per-instance copy; bitwise rbws_fn_apply's result) */
int rbws_fn_apply_shared(int count, int nterms, int c, const double* theta, const double* coef,
                         const double* x, const double* b, double* y, int mode, void* stream);
/* doubles of the band factors: planar = 1 z-plane blocks (PlaneSmootherPair,
 * multigrid.py:56-77: splu of A[plane, plane]), planar = 0 the whole level (coarsest
 * factor, multigrid.py:154-168: cho_factor) */
int64_t rbws_fn_band_doubles(int count, int c, int planar);
/* build + banded Cholesky of every block (info[sys] = first bad pivot + 1, or 0) */
int rbws_fn_band_factor(int count, int c, int planar, const double* coefA, double* band,
                        int* info, void* stream);
/* block solves of r (overwritten): mode 0 x = A_blk^-1 r, mode 1 x += omega A_blk^-1 r
 * (plane-Jacobi sweep, multigrid.py:91-95; cho_solve, multigrid.py:216) */
int rbws_fn_band_solve(int count, int c, int planar, const double* band, double* r, double* x,
                       double omega, int mode, void* stream);
/* The band factor transposed (bandT[i][d] = L[i+d][i], the columns of L as rows), for the
 * scatter-form forward substitution of rbws_fn_band_solve_t; same size as the band. */
int rbws_fn_band_transpose(int count, int c, int planar, const double* band, double* bandT,
                           void* stream);
/* rbws_fn_band_solve with both substitutions in scatter form (rows of bandT forward, rows of
 * band backward), one warp per system, rows owned round-robin by the lanes: no dot-product
 * reduction on the dependency chain.  Same arguments and results (up to rounding). */
int rbws_fn_band_solve_t(int count, int c, int planar, const double* band, const double* bandT,
                         double* r, double* x, double omega, int mode, void* stream);
/* one block Gauss-Seidel sweep over the z-planes of x (ascending if forward, else
 * descending): x_p = A_pp^-1 (b_p - A[p,p-1] x_{p-1} - A[p,p+1] x_{p+1}) with the plane
 * factors of rbws_fn_band_factor(planar = 1); scratch >= count (c+1)^2 doubles —
 * PlaneSmootherPair._sweep (multigrid.py:79-89), smoother "plane-z" */
int rbws_fn_plane_gs_sweep(int count, int c, const double* coefA, const double* band,
                           const double* b, double* x, double* scratch, int forward, void* stream);
/* b = P^T r (cc coarse cells; zero on coarse Dirichlet nodes) — grid.py:131-141 */
int rbws_fn_restrict(int count, int cc, const double* r_fine, double* b_coarse,
                     const unsigned char* coarse_mask, void* stream);
/* u += P e on fine free nodes — multigrid.py:220 */
int rbws_fn_prolong_add(int count, int cc, const double* e_coarse, double* u_fine,
                        const unsigned char* fine_mask, void* stream);
/* x += omega r / diag(A) on free nodes — damped point Jacobi, kernels.py:98-115 */
int rbws_fn_point_jacobi(int count, int c, const double* coefA, const double* r, double* x,
                         double omega, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RBWS_B200_H */
