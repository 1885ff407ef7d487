// Slab-decomposed MGCG for one large instance (BASELINE configs[4]).
#pragma once

#include <array>
#include <vector>

#include "comm.cuh"
#include "solver.cuh"

namespace rbws {

// vectors of one slab on one level
enum SlabVec : int {
  SV_X = 0, SV_F, SV_R, SV_P, SV_P2, SV_S,  // finest level: PCG state
  SV_T,                                      // smoother scratch / true residual
  SV_DINV,                                   // 1/diag (finest level: with halo planes)
  SV_B, SV_E, SV_U,                          // distributed coarse levels: rhs, correction, w D^-1 b
  SV_N
};

// One slab: global planes [k0, k1) of every distributed level, stored as the
// planes k0-1 .. k1 (halo planes at both ends) plus a two-plane zero tail.
struct SlabPart {
  int rank = 0;                                 // global slab index
  std::vector<int> k0, k1;                      // per level (distributed levels only)
  std::vector<std::array<double*, SV_N>> v;     // per level buffer base pointers (plane k0-1)
};

struct Slab {
  Hierarchy* h = nullptr;
  int R = 1;          // slabs in the whole job
  int nloc = 1;       // slabs held by this process (consecutive global indices)
  int first = 0;      // global index of the first local slab
  int L = 0;          // levels
  int Ld = 0;         // levels Ld .. L-1 are slab-distributed, 0 .. Ld-1 replicated
  double omega = 0.7;
  Comm* comm = nullptr;  // inter-process transport (null: all slabs in this process)
  Batch* rep = nullptr;  // replicated coarse levels (a batch of one, levels < Ld)
  std::vector<SlabPart> parts;
  double* theta = nullptr;
  // PCG scalars of the instance (every process holds identical copies)
  double *partial = nullptr, *partial2 = nullptr, *rs = nullptr, *alpha = nullptr,
         *beta = nullptr, *scale = nullptr, *tres = nullptr, *hist = nullptr;
  int *active = nullptr, *iters = nullptr, *status = nullptr, *nactive = nullptr;
  int* h_nactive = nullptr;
  int tiles = 0, vtiles = 0, ftiles = 0, hist_len = 0;
  bool ready = false;

  ~Slab();
  int cells(int l) const { return h->cells[l]; }
  double* V(const SlabPart& p, int l, int vid) const;  // virtual base: plane k at V + k n^2
  LaunchCtx lc(const SlabPart& p, int l, cudaStream_t s, bool act) const;
  int xchg(int l, int vid, int dirs, cudaStream_t s);
  int gather_partials(double* part, int tiles_per_slab, cudaStream_t s);
  int vcycle(int l, int vb, int vout, bool dot, cudaStream_t s);
};

enum : int { XCHG_UP = 1, XCHG_DOWN = 2, XCHG_BOTH = 3 };

int slab_create(Slab** out, Hierarchy* h, int nslabs, int first, int nloc, Comm* comm,
                double omega);
int slab_setup(Slab* s, const double* theta, int* n_bad, cudaStream_t stream);
// copy global planes [p0, p0+planes) of src (one padded instance region, device or host) into
// the owned planes of vector vid (SV_X or SV_F); store: owned planes of SV_X into dst
int slab_load(Slab* s, int vid, const double* src, int64_t p0, int planes, cudaStream_t stream);
int slab_store(Slab* s, int vid, double* dst, int64_t p0, int planes, cudaStream_t stream);
// x = P ec: warm start prolonged from a full coarse vector (n/2 cells, one instance)
int slab_prolong_x(Slab* s, const double* ec, cudaStream_t stream);
int slab_solve(Slab* s, double delta, int l_max, int* iters, double* hist, double* true_res,
               int* status, cudaStream_t stream);

}  // namespace rbws
