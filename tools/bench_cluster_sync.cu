// bench_cluster_sync.cu -- cycles of the synchronisation primitives the projection kernel is
// built from, on one 512-thread CTA per SM: __syncthreads, cluster.sync at 2..16 CTAs, and
// the cluster_combine pattern (DSMEM stores into every CTA + cluster.sync + butterfly).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bench_cluster_sync \
//        tools/bench_cluster_sync.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

constexpr int REPS = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
               "d"(v), "r"(rbar) : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(su32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ double wtree(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_sync(long long* out, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[2][16][4];
  __shared__ uint64_t mb[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int cs = (int)cl.num_blocks();
  const unsigned rank = cl.block_rank();
  double acc = threadIdx.x;
  cl.sync();
  const long long t0 = clock64();
  for (int r = 0; r < REPS; ++r) {
    if (mode == 0) {
      __syncthreads();
    } else if (mode == 1) {
      cl.sync();
    } else if (mode == 2) {  // cluster_combine of 2 values
      if ((int)threadIdx.x < cs) {
        double* dst = cl.map_shared_rank(&slot[r & 1][0][0], (int)threadIdx.x);
        dst[rank * 4 + 0] = acc;
        dst[rank * 4 + 1] = acc + 1.0;
      }
      cl.sync();
      const int lane = threadIdx.x & 31;
      double x = lane < cs ? slot[r & 1][lane][0] : 0.0;
      for (int o = 1; o < cs; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      acc += x * 1e-30;
    } else if (mode == 4) {  // st.async of 2 values into every CTA, mbarrier wait
      const int b = r & 1;
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[b])),
                     "r"(cs * 16) : "memory");
      if ((int)threadIdx.x < cs) {
        const uint32_t ra = mapa(su32(&slot[b][rank][0]), (int)threadIdx.x);
        const uint32_t rb = mapa(su32(&mb[b]), (int)threadIdx.x);
        st_async_f64(ra, acc, rb);
        st_async_f64(ra + 8, acc + 1.0, rb);
      }
      wait_par(&mb[b], (uint32_t)((r >> 1) & 1));
      const int lane = threadIdx.x & 31;
      double x = lane < cs ? slot[b][lane][0] : 0.0;
      for (int o = 1; o < cs; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      acc += x * 1e-30;
    } else if (mode == 5 || mode == 6) {  // block reduce of 5 doubles (project.cu block_reduce)
      __shared__ double wv[2][16][6];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      double v[5] = {acc, acc + 1, acc + 2, acc + 3, acc + 4};
      const int kinds[5] = {0, 1, 1, 2, 2};
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const double x = kinds[c] == 1 ? wmax(v[c]) : wtree(v[c]);
        if (lane == 0) wv[r & 1][warp][c] = x;
      }
      __syncthreads();
      if (mode == 5) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double x = lane < 16 ? wv[r & 1][lane][c] : 0.0;
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = kinds[c] == 1 ? fmax(x, y) : __dadd_rn(x, y);
          }
          v[c] = __shfl_sync(0xffffffffu, x, 0);
        }
      }
      acc += (v[0] + v[1] + v[2] + v[3] + v[4]) * 1e-30;
    } else if (mode == 7) {  // one warp tree of one double
      acc += wtree(acc) * 1e-30;
    } else if (mode == 3) {  // barrier.cluster arrive.relaxed + wait (no fence)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / REPS;
  cl.sync();  // no CTA exits while st.async into it may be in flight
  if (acc == -1.0) out[1] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const char* names[8] = {"__syncthreads", "cluster.sync", "cluster_combine(2)", "barrier.cluster relaxed",
                          "st.async combine(2)", "block_reduce<5>", "block_reduce<5> 1st half", "warp_tree(1)"};
  for (int mode = 0; mode < 8; ++mode) {
    for (int cs : {1, 2, 4, 8, 16}) {
      if ((mode == 0 || mode >= 5) && cs > 1) continue;
      cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1, 1);
      cfg.blockDim = dim3(512, 1, 1);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      long long cyc = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaLaunchKernelEx(&cfg, k_sync, d, mode);
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      }
      cudaError_t e = cudaGetLastError();
      std::printf("%-26s cluster %2d: %lld cycles per call%s\n", names[mode], cs, cyc,
                  e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
