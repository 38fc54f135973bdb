// stream_bench2.cu -- which factor slows the GEMV pipeline: access order, copy size, or
// consumer work?  Same 3 x 64 KB TMA ring as gemv.cu, one CTA (1 producer + 4 consumer
// warps) per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o sb2 tools/stream_bench2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
template <int N, class F>
__device__ __forceinline__ double2 tree2(const F& leaf, int base = 0) {
  if constexpr (N == 1) {
    return leaf(base);
  } else {
    const double2 a = tree2<N / 2>(leaf, base);
    const double2 b = tree2<N / 2>(leaf, base + N / 2);
    return make_double2(add(a.x, b.x), add(a.y, b.y));
  }
}

constexpr int STAGES = 3;
constexpr int SB = 65536;

// order 0: CTA c reads chunks c, c+G, ... (contiguous 64 KB chunks)
// order 1: adjoint order: task t = (cg = t / nrr, rr = t % nrr), 16 stages per task, stage s =
//          row block rr*16+s, chunk at (rb * ncb + 4 cg) * 16 KB   (ncb = 512, nrb = 256)
// pieces: number of bulk copies per stage; heavy: tree compute like the adjoint consumer
__global__ void __launch_bounds__(160, 1) k(const char* src, int order, int pieces, int heavy,
                                            double* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = (uint64_t*)(sm + STAGES * SB);
  uint64_t* empty = full + STAGES;
  __shared__ double rs[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) rs[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  const int ntasks = 2048, nst = 16;
  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int cg = t / 16, rr = t % 16;
        for (int s = 0; s < nst; ++s) {
          int64_t off;
          if (order == 0) off = ((int64_t)t * nst + s) * SB;
          else off = ((int64_t)(rr * 16 + s) * 512 + 4 * cg) * 16384;
          waitp(&empty[st], ph ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                       "r"(SB)
                       : "memory");
          const int piece = SB / pieces;
          for (int o = 0; o < SB; o += piece)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(sm + st * SB + o)),
                "l"(src + off + o), "r"(piece), "r"(su32(&full[st]))
                : "memory");
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  double acc = 0.0;
  int st = 0;
  uint32_t ph = 0;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    for (int s = 0; s < nst; ++s) {
      waitp(&full[st], ph);
      const double2* ku = (const double2*)(sm + st * SB + cw * 16384);
      if (heavy) {
        double2 v = tree2<32>([&](int i) {
          const double2 kk = ku[i * 32 + (lane ^ (i & 7))];
          const double r = rs[i];
          return make_double2(mul(kk.x, r), mul(kk.y, r));
        });
        acc = add(acc, add(v.x, v.y));
      } else {
        for (int i = lane; i < 1024; i += 32) acc += ku[i].x;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
      if (++st == STAGES) {
        st = 0;
        ph ^= 1u;
      }
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const int64_t bytes = 2LL << 30;
  char* src;
  double* out;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(src, 0, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = STAGES * SB + 64;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int order = 0; order < 2; ++order)
    for (int pieces : {1, 4})
      for (int heavy = 0; heavy < 2; ++heavy) {
        for (int w = 0; w < 2; ++w) k<<<sms, 160, smem>>>(src, order, pieces, heavy, out);
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 5; ++r) k<<<sms, 160, smem>>>(src, order, pieces, heavy, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("order=%s pieces=%d consumer=%s : %7.1f GB/s\n", order ? "adjoint" : "linear",
               pieces, heavy ? "tree  " : "light ", 5.0 * bytes / (ms / 1e3) / 1e9);
      }
  return 0;
}
