// NCCL communicator of the multi-GPU kNN layouts, owned by the library so the
// per-round histogram all-reduce and the result all-gather + exact merge run without any host
// language in the loop. NCCL is loaded at run time (dlopen): the library itself never requires
// it, and inside a process that already loaded NCCL (e.g. through torch) the same copy is used,
// so every rank of a job runs one NCCL version. Only the types come from <nccl.h>.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "knn.cuh"

namespace mihg {

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

template <typename F>
void bind(void* so, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(so, name));
  if (!fn) throw NcclError(std::string("NCCL symbol missing: ") + name);
}

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string load_error;
  std::call_once(once, [] {
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process
    if (!so) {
      if (const char* p = std::getenv("MIHG_NCCL_LIBRARY")) so = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!so) {
      load_error = std::string("cannot load NCCL (libnccl.so.2): ") + (dlerror() ? dlerror() : "?");
      return;
    }
    try {
      bind(so, "ncclGetUniqueId", api.get_unique_id);
      bind(so, "ncclCommInitRank", api.comm_init_rank);
      bind(so, "ncclCommDestroy", api.comm_destroy);
      bind(so, "ncclAllReduce", api.all_reduce);
      bind(so, "ncclAllGather", api.all_gather);
      bind(so, "ncclGetErrorString", api.error_string);
      bind(so, "ncclGetVersion", api.get_version);
      api.so = so;
    } catch (const std::exception& e) {
      load_error = e.what();
    }
  });
  if (!api.so) throw NcclError(load_error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct Comm {
  ncclComm_t c = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

void comm_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
}

Comm* comm_init(const uint8_t* id128, int nranks, int rank, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("comm: need 0 <= rank < nranks");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  MIHG_CUDA(cudaSetDevice(device));
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  const ncclResult_t r = nccl().comm_init_rank(&c->c, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  return c;
}

void comm_free(Comm* c) {
  if (!c) return;
  if (c->c) nccl().comm_destroy(c->c);
  delete c;
}

int comm_size(const Comm* c) { return c->nranks; }
int comm_rank(const Comm* c) { return c->rank; }
int nccl_version() {
  int v = 0;
  nccl_check(nccl().get_version(&v), "ncclGetVersion");
  return v;
}

// In-place sum of n elements (dtype 0: u32, 1: u64) across the communicator, on `st`.
void comm_allreduce_sum(Comm* c, void* ptr, uint64_t n, int dtype, cudaStream_t st) {
  nccl_check(nccl().all_reduce(ptr, ptr, n, dtype == 0 ? ncclUint32 : ncclUint64, ncclSum, c->c, st),
             "ncclAllReduce");
}

// recv[rank * bytes ...] <- every rank's `bytes` bytes of send, on `st`.
void comm_allgather(Comm* c, const void* send, void* recv, uint64_t bytes, cudaStream_t st) {
  nccl_check(nccl().all_gather(send, recv, bytes, ncclUint8, c->c, st), "ncclAllGather");
}

}  // namespace mihg
