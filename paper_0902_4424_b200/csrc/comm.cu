// comm.cu -- NCCL transport of the column-sharded solver.
//
// Rank r of R holds K[:, r*p/R : (r+1)*p/R]; per iteration the ranks exchange two vectors
// with ncclAllGather on the solver stream (captured into the iteration graph): the shard
// tree values of K d (n doubles per rank) and of K^T r (p/R doubles per rank).  NCCL is
// loaded at run time (the libnccl.so.2 torch already mapped, else the system one), so the
// library has no link-time NCCL dependency and single-GPU use never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "comm.h"
#include "engine.h"

namespace l1g {

namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("L1G_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if (n && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      a.err = "NCCL runtime (libnccl.so.2) not found";
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather &&
           a.group_start && a.group_end;
    if (!a.ok) a.err = "NCCL runtime lacks the expected entry points";
  });
  if (!a.ok) throw RuntimeFailure(a.err);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* m = api().error_string ? api().error_string(r) : "?";
  throw RuntimeFailure(std::string(what) + ": " + m);
}
}  // namespace

static_assert(sizeof(ncclUniqueId) == kCommIdBytes, "NCCL unique id size");

void comm_unique_id(void* out) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

Comm* comm_create(int device, int rank, int nranks, const void* id_bytes) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("comm: bad rank / size");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  L1G_CUDA_HOST(cudaSetDevice(device));
  auto* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclComm_t h = nullptr;
  try {
    check(api().comm_init_rank(&h, nranks, id, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  c->handle = h;
  return c;
}

Comm* comm_create_host(int device, int rank, int nranks, HostAllgatherFn fn, void* user) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("comm: bad rank / size");
  if (!fn) throw InvalidArgument("comm: host transport needs an allgather function");
  auto* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  c->host_fn = fn;
  c->host_user = user;
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->handle) api().comm_destroy(static_cast<ncclComm_t>(c->handle));
  delete c;
}

void comm_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t s) {
  check(api().all_gather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(c->handle), s),
        "ncclAllGather");
}

// several allgathers as one NCCL group (one launch; the pieces of a shard's packet)
void comm_allgather_group(Comm* c, int n, const double* const* send, double* const* recv,
                          const size_t* count, cudaStream_t s) {
  NcclApi& a = api();
  check(a.group_start(), "ncclGroupStart");
  for (int i = 0; i < n; ++i) {
    const ncclResult_t r = a.all_gather(send[i], recv[i], count[i], ncclFloat64,
                                        static_cast<ncclComm_t>(c->handle), s);
    if (r != ncclSuccess) {
      a.group_end();
      check(r, "ncclAllGather");
    }
  }
  check(a.group_end(), "ncclGroupEnd");
}

}  // namespace l1g
