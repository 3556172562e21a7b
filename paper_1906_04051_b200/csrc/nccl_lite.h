// Minimal runtime binding to NCCL (dlopen of libnccl.so.2).  The multi-GPU
// path needs five entry points; binding them at run time keeps libpgmres free
// of a link-time NCCL dependency and lets it share the libnccl that
// torch.distributed already loaded in the process (same soname).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstddef>
#include <cstring>

namespace nccl_lite {

struct UniqueId {
  char internal[128];
};
typedef int (*fn_init)(void** comm, int nranks, UniqueId id, int rank);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_p2p)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_recv)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_void)();
typedef int (*fn_destroy)(void*);
typedef int (*fn_getid)(UniqueId*);
typedef int (*fn_allgather)(const void*, void*, size_t, int, void*, cudaStream_t);

struct Api {
  void* h = nullptr;
  fn_init init = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_p2p send = nullptr;
  fn_recv recv = nullptr;
  fn_void gstart = nullptr, gend = nullptr;
  fn_destroy destroy = nullptr;
  fn_getid getid = nullptr;
  fn_allgather allgather = nullptr;
  bool ok = false;
};

inline Api& api() {
  static Api a = [] {
    Api x;
    x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) return x;
    x.init = (fn_init)dlsym(x.h, "ncclCommInitRank");
    x.allreduce = (fn_allreduce)dlsym(x.h, "ncclAllReduce");
    x.send = (fn_p2p)dlsym(x.h, "ncclSend");
    x.recv = (fn_recv)dlsym(x.h, "ncclRecv");
    x.gstart = (fn_void)dlsym(x.h, "ncclGroupStart");
    x.gend = (fn_void)dlsym(x.h, "ncclGroupEnd");
    x.destroy = (fn_destroy)dlsym(x.h, "ncclCommDestroy");
    x.getid = (fn_getid)dlsym(x.h, "ncclGetUniqueId");
    x.allgather = (fn_allgather)dlsym(x.h, "ncclAllGather");
    x.ok = x.init && x.allreduce && x.send && x.recv && x.gstart && x.gend && x.destroy;
    return x;
  }();
  return a;
}

constexpr int kFloat64 = 8;  // ncclFloat64
constexpr int kSum = 0;      // ncclSum

inline bool available() { return api().ok; }
inline int comm_init_rank(void** comm, int world, const void* id, int rank) {
  UniqueId u;
  std::memcpy(u.internal, id, sizeof(u.internal));
  return api().init(comm, world, u, rank);
}
inline int allreduce_sum_f64(const double* in, double* out, size_t n, void* comm, cudaStream_t s) {
  return api().allreduce(in, out, n, kFloat64, kSum, comm, s);
}
inline int send_f64(const double* p, size_t n, int peer, void* comm, cudaStream_t s) {
  return api().send(p, n, kFloat64, peer, comm, s);
}
inline int recv_f64(double* p, size_t n, int peer, void* comm, cudaStream_t s) {
  return api().recv(p, n, kFloat64, peer, comm, s);
}
// deterministic mode: every rank's plane partials to every rank
inline int allgather_f64(const double* in, double* out, size_t n_per_rank, void* comm,
                         cudaStream_t s) {
  if (!api().allgather) return 1;
  return api().allgather(in, out, n_per_rank, kFloat64, comm, s);
}
inline int group_start() { return api().gstart(); }
inline int group_end() { return api().gend(); }
inline int comm_destroy(void* c) { return api().destroy(c); }
inline int get_unique_id(void* out128) {
  if (!api().getid) return -1;
  UniqueId u;
  const int rc = api().getid(&u);
  std::memcpy(out128, u.internal, sizeof(u.internal));
  return rc;
}

}  // namespace nccl_lite
