// bench_round.cu -- cycles of the projection's synchronisation rounds on a 16-CTA cluster
// of 512 threads: cluster barrier alone, block reduction alone, block + cluster reduction.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -o tools/bench_round tools/bench_round.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
namespace cg = cooperative_groups;

constexpr int PT = 512, PW = 16;
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
struct Sh {
  double wv[2][PW][4];
  double slot[2][16][4];
  unsigned long long bar[2];
};
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(PT, 1) k_round(int mode, int R, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ Sh sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned rank = cl.block_rank();
  const int cs = 16;
  double v0 = threadIdx.x * 1e-3, v1 = rank;
  int pb = 0, pc = 0;
  unsigned ph = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sh.bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  const long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
    if (mode == 0) {
      cl.sync();
    } else if (mode == 4) {
      __syncthreads();
    } else {
      double x0 = warp_tree(v0), x1 = warp_tree(v1);
      if (lane == 0) {
        sh.wv[pb][warp][0] = x0;
        sh.wv[pb][warp][1] = x1;
      }
      __syncthreads();
      double y0 = lane < PW ? sh.wv[pb][lane][0] : 0.0, y1 = lane < PW ? sh.wv[pb][lane][1] : 0.0;
#pragma unroll
      for (int o = 1; o < PW; o <<= 1) {
        y0 = add(y0, __shfl_xor_sync(0xffffffffu, y0, o));
        y1 = add(y1, __shfl_xor_sync(0xffffffffu, y1, o));
      }
      y0 = __shfl_sync(0xffffffffu, y0, 0);
      y1 = __shfl_sync(0xffffffffu, y1, 0);
      pb ^= 1;
      if (mode == 5) {  // st.async into every CTA's slots, completion on its mbarrier
        if (threadIdx.x == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sh.bar[pc])),
                       "r"(cs * 16) : "memory");
        if ((int)threadIdx.x < cs) {
          const unsigned ra = mapa(smem_u32(&sh.slot[pc][rank][0]), threadIdx.x);
          const unsigned rb = mapa(smem_u32(&sh.bar[pc]), threadIdx.x);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                       "d"(y0), "d"(y1), "r"(rb) : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
            "@P1 bra DONE_%=;\n\t"
            "bra WAIT_%=;\n"
            "DONE_%=:\n\t}" ::"r"(smem_u32(&sh.bar[pc])), "r"((ph >> pc) & 1u) : "memory");
        ph ^= 1u << pc;
        double z0 = lane < cs ? sh.slot[pc][lane][0] : 0.0, z1 = lane < cs ? sh.slot[pc][lane][1] : 0.0;
        for (int o = 1; o < cs; o <<= 1) {
          z0 = add(z0, __shfl_xor_sync(0xffffffffu, z0, o));
          z1 = add(z1, __shfl_xor_sync(0xffffffffu, z1, o));
        }
        y0 = __shfl_sync(0xffffffffu, z0, 0);
        y1 = __shfl_sync(0xffffffffu, z1, 0);
        pc ^= 1;
      }
      if (mode == 2 || mode == 3) {
        if ((int)threadIdx.x < cs) {
          Sh* dst = cl.map_shared_rank(&sh, (int)threadIdx.x);
          dst->slot[pc][rank][0] = y0;
          dst->slot[pc][rank][1] = y1;
        }
        if (mode == 2) {
          cl.sync();
        } else {  // split barrier with explicit release / acquire
          asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
          asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        }
        double z0 = lane < cs ? sh.slot[pc][lane][0] : 0.0, z1 = lane < cs ? sh.slot[pc][lane][1] : 0.0;
        for (int o = 1; o < cs; o <<= 1) {
          z0 = add(z0, __shfl_xor_sync(0xffffffffu, z0, o));
          z1 = add(z1, __shfl_xor_sync(0xffffffffu, z1, o));
        }
        y0 = __shfl_sync(0xffffffffu, z0, 0);
        y1 = __shfl_sync(0xffffffffu, z1, 0);
        pc ^= 1;
      }
      v0 = add(v0, y0 * 1e-30);
      v1 = add(v1, y1 * 1e-30);
    }
  }
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && rank == 0) {
    out[0] = (t1 - t0) / R;
    out[1] = (long long)(v0 + v1);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k_round, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[6] = {"cluster.sync only", "block reduce (2 values)", "block + cluster (cg sync)",
                          "block + cluster (arrive.release/wait.acquire)", "__syncthreads only", "block + cluster (st.async + mbarrier)"};
  for (int mode = 0; mode < 6; ++mode) {
    long long h[2];
    for (int rep = 0; rep < 3; ++rep) k_round<<<16, PT>>>(mode, 200, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    std::printf("%-48s %lld cycles/round, value %lld (%s)\n", names[mode], h[0], h[1], cudaGetErrorString(e));
  }
  return 0;
}
