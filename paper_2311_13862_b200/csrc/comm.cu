// NCCL transport for the slab-decomposed solver (see comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.cuh"

int rbws_set_error(const char* msg, const char* file, int line);
#define RBWS_FAIL(msg) return rbws_set_error(msg, __FILE__, __LINE__)

namespace rbws {

namespace {

struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the libnccl already mapped into the process (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define RBWS_SYM(f, name) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, name))
    RBWS_SYM(get_id, "ncclGetUniqueId");
    RBWS_SYM(init, "ncclCommInitRank");
    RBWS_SYM(destroy, "ncclCommDestroy");
    RBWS_SYM(group_start, "ncclGroupStart");
    RBWS_SYM(group_end, "ncclGroupEnd");
    RBWS_SYM(send, "ncclSend");
    RBWS_SYM(recv, "ncclRecv");
    RBWS_SYM(allgather, "ncclAllGather");
    RBWS_SYM(errstr, "ncclGetErrorString");
#undef RBWS_SYM
    a.ok = a.get_id && a.init && a.destroy && a.group_start && a.group_end && a.send &&
           a.recv && a.allgather && a.errstr;
  });
  return a;
}

int nccl_fail(ncclResult_t r, const char* file, int line) {
  const NcclApi& a = api();
  return rbws_set_error(a.errstr ? a.errstr(r) : "NCCL error", file, line);
}

}  // namespace

#define RBWS_NCCL(expr)                                                   \
  do {                                                                    \
    ncclResult_t _r = (expr);                                             \
    if (_r != ncclSuccess) return nccl_fail(_r, __FILE__, __LINE__);      \
  } while (0)
#define RBWS_NEED_NCCL() \
  if (!api().ok) RBWS_FAIL("libnccl.so.2 not found (needed for multi-process slabs)")

Comm::~Comm() {
  if (nccl && api().ok) api().destroy(reinterpret_cast<ncclComm_t>(nccl));
}

int comm_unique_id(unsigned char* out) {
  RBWS_NEED_NCCL();
  ncclUniqueId id;
  RBWS_NCCL(api().get_id(&id));
  static_assert(sizeof(id) == kCommIdBytes, "NCCL unique id size");
  memcpy(out, &id, sizeof(id));
  return 0;
}

int comm_create(Comm** out, const unsigned char* id, int nprocs, int rank) {
  RBWS_NEED_NCCL();
  if (nprocs < 1 || rank < 0 || rank >= nprocs) RBWS_FAIL("bad communicator rank / size");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c;
  RBWS_NCCL(api().init(&c, nprocs, uid, rank));
  Comm* cm = new Comm();
  cm->nccl = c;
  cm->nprocs = nprocs;
  cm->rank = rank;
  *out = cm;
  return 0;
}

int comm_group_start() {
  RBWS_NEED_NCCL();
  RBWS_NCCL(api().group_start());
  return 0;
}

int comm_group_end() {
  RBWS_NEED_NCCL();
  RBWS_NCCL(api().group_end());
  return 0;
}

int comm_send(Comm* c, const double* buf, size_t count, int peer, cudaStream_t s) {
  RBWS_NCCL(api().send(buf, count, ncclDouble, peer, reinterpret_cast<ncclComm_t>(c->nccl), s));
  return 0;
}

int comm_recv(Comm* c, double* buf, size_t count, int peer, cudaStream_t s) {
  RBWS_NCCL(api().recv(buf, count, ncclDouble, peer, reinterpret_cast<ncclComm_t>(c->nccl), s));
  return 0;
}

int comm_allgather(Comm* c, double* buf, size_t count, cudaStream_t s) {
  RBWS_NCCL(api().allgather(buf + (size_t)c->rank * count, buf, count, ncclDouble,
                            reinterpret_cast<ncclComm_t>(c->nccl), s));
  return 0;
}

}  // namespace rbws
