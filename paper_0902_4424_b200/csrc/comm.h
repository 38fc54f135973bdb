// comm.h -- NCCL transport of the column-sharded solver (comm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>

namespace l1g {

constexpr int kCommIdBytes = 128;  // ncclUniqueId

// host allgather of the host transport: recv[r * count + i] = rank r's send[i]
typedef int (*HostAllgatherFn)(const double* send, double* recv, int64_t count, void* user);

struct Comm {
  void* handle = nullptr;  // ncclComm_t (NCCL transport)
  int rank = 0, nranks = 1, device = 0;
  // host transport (no NCCL): the exchanges stage through pinned host memory and a
  // caller-supplied allgather (e.g. gloo), run as host nodes of the iteration graphs
  HostAllgatherFn host_fn = nullptr;
  void* host_user = nullptr;
  bool host() const { return host_fn != nullptr; }
};

void comm_unique_id(void* out);
Comm* comm_create(int device, int rank, int nranks, const void* id_bytes);
Comm* comm_create_host(int device, int rank, int nranks, HostAllgatherFn fn, void* user);
void comm_destroy(Comm* c);
void comm_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t s);
void comm_allgather_group(Comm* c, int n, const double* const* send, double* const* recv,
                          const size_t* count, cudaStream_t s);

}  // namespace l1g

#define L1G_CUDA_HOST(call)                                                             \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess) throw ::l1g::CudaError(e__, #call, __FILE__, __LINE__);     \
  } while (0)
