// Inter-process transport of the slab-decomposed solver (slab.cu): NCCL
// point-to-point halo planes and all-gathers of dot-product partials, issued on
// the solver's stream.  libnccl is opened at run time (dlopen), so the library
// loads on hosts without NCCL and shares the copy torch.distributed already
// loaded when there is one.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace rbws {

constexpr int kCommIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int nprocs = 1, rank = 0;
  ~Comm();
};

// rank 0 creates the id; every rank passes the same bytes to comm_create
int comm_unique_id(unsigned char* out);
int comm_create(Comm** out, const unsigned char* id, int nprocs, int rank);

// grouped halo traffic: sends/recvs between comm_group_start/comm_group_end
int comm_group_start();
int comm_group_end();
int comm_send(Comm* c, const double* buf, size_t count, int peer, cudaStream_t s);
int comm_recv(Comm* c, double* buf, size_t count, int peer, cudaStream_t s);
// in place: buf + rank*count is this rank's chunk
int comm_allgather(Comm* c, double* buf, size_t count, cudaStream_t s);

}  // namespace rbws
