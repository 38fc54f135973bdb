// stream_bench.cu -- how fast can one kernel stream a 2 GiB fp64 array on this B200?
// Compares plain LDG.128 streaming with cp.async.bulk (TMA engine) multi-stage rings of
// different depths / stage sizes, 1 or 2 CTAs per SM.  Used to choose the GEMV pipeline.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void ldg_kernel(const double2* __restrict__ a, int64_t n2, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n2; i += 8 * stride) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) acc += a[i].x;
  if (acc == 1.2345) out[0] = acc;
}

template <int STAGES>
__global__ void __launch_bounds__(160) tma_kernel(const char* src, int64_t total, int64_t stage_bytes,
                                                  double* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = (uint64_t*)(sm + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nchunks = total / stage_bytes;
  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
                su32(&empty[st])),
            "r"(ph ^ 1u)
            : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                     "r"((uint32_t)stage_bytes)
                     : "memory");
        const int64_t piece = stage_bytes >= 16384 ? 16384 : stage_bytes;
        for (int64_t o = 0; o < stage_bytes; o += piece)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(sm + st * stage_bytes + o)),
              "l"(src + c * stage_bytes + o), "r"((uint32_t)piece), "r"(su32(&full[st]))
              : "memory");
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  double acc = 0.0;
  int st = 0;
  uint32_t ph = 0;
  const int cw = warp - 1;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
            su32(&full[st])),
        "r"(ph)
        : "memory");
    const double2* p = (const double2*)(sm + st * stage_bytes);
    const int64_t n16 = stage_bytes / 16;
    for (int64_t i = cw * 32 + lane; i < n16; i += 128) {
      double2 v = p[i];
      acc += v.x * v.y;
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
    if (++st == STAGES) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int STAGES>
int run_tma(const char* src, int64_t bytes, int64_t stage_bytes, int ctas_per_sm, int sms,
            double* out, cudaEvent_t e0, cudaEvent_t e1) {
  const size_t smem = STAGES * stage_bytes + 2 * STAGES * 8;
  CK(cudaFuncSetAttribute(tma_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = sms * ctas_per_sm;
  for (int w = 0; w < 2; ++w) tma_kernel<STAGES><<<grid, 160, smem>>>(src, bytes, stage_bytes, out);
  CK(cudaEventRecord(e0));
  const int R = 5;
  for (int r = 0; r < R; ++r) tma_kernel<STAGES><<<grid, 160, smem>>>(src, bytes, stage_bytes, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("TMA stages=%2d stage=%6lld B ctas/SM=%d smem=%7zu : %7.1f GB/s\n", STAGES,
         (long long)stage_bytes, ctas_per_sm, smem, R * bytes / (ms / 1e3) / 1e9);
  return 0;
}

int main() {
  const int64_t bytes = 2LL << 30;
  char* src;
  double* out;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(src, 1, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int k : {2, 4, 8}) {
    for (int w = 0; w < 2; ++w) ldg_kernel<<<sms * k, 512>>>((const double2*)src, bytes / 16, out);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) ldg_kernel<<<sms * k, 512>>>((const double2*)src, bytes / 16, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("LDG  blocks/SM=%d x512 unroll8           : %7.1f GB/s\n", k, 5 * bytes / (ms / 1e3) / 1e9);
  }
  run_tma<3>(src, bytes, 65536, 1, sms, out, e0, e1);
  run_tma<6>(src, bytes, 32768, 1, sms, out, e0, e1);
  run_tma<12>(src, bytes, 16384, 1, sms, out, e0, e1);
  run_tma<24>(src, bytes, 8192, 1, sms, out, e0, e1);
  run_tma<3>(src, bytes, 32768, 2, sms, out, e0, e1);
  run_tma<6>(src, bytes, 16384, 2, sms, out, e0, e1);
  run_tma<12>(src, bytes, 8192, 2, sms, out, e0, e1);
  run_tma<4>(src, bytes, 16384, 3, sms, out, e0, e1);
  run_tma<2>(src, bytes, 32768, 3, sms, out, e0, e1);
  run_tma<8>(src, bytes, 4096, 4, sms, out, e0, e1);
  return 0;
}
