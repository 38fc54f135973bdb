// comm.h -- NCCL transport of the column-sharded solver (comm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>

namespace l1g {

constexpr int kCommIdBytes = 128;  // ncclUniqueId

struct Comm {
  void* handle = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1, device = 0;
};

void comm_unique_id(void* out);
Comm* comm_create(int device, int rank, int nranks, const void* id_bytes);
void comm_destroy(Comm* c);
void comm_allgather(Comm* c, const double* send, double* recv, size_t count, cudaStream_t s);

}  // namespace l1g

#define L1G_CUDA_HOST(call)                                                             \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess) throw ::l1g::CudaError(e__, #call, __FILE__, __LINE__);     \
  } while (0)
