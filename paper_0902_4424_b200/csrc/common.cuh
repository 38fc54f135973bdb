// common.cuh -- shared device helpers for the B200 GPSS engine (sm_100a only).
//
// Numerics contract: every product is rounded (no FMA; the
// library is compiled with -fmad=false and the hot paths spell __dmul_rn/__dadd_rn), and
// every sum is the pairwise sum with power-of-two splits over the element index.  The CPU
// oracle (oracle/l1oracle.c) implements the same order, so results agree bit for bit.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <mutex>

#ifndef __CUDACC__
#error "common.cuh is CUDA-only"
#endif

namespace l1g {

// ---- K tile layout ------------------------------------------------------------------
// K (n x p, fp64) is stored as 32 x 64 tiles, tile (rb, cb) at ((rb * NCB) + cb) * 2048
// doubles.  Inside a tile each column is one contiguous 256-byte run of its 32 rows, with
// the rows XOR-swizzled by the column pair: element (i, j) at j*32 + (i ^ ((j >> 1) & 15)).
// Shared-memory reads are conflict-free for both dense patterns (lanes = rows at a fixed
// column for the forward product, lanes = column pairs at a fixed row for the adjoint), and
// one column of a tile is a single coalesced 256-byte global read, which is what the
// support-sparse forward product gathers.
constexpr int TR = 32;
constexpr int TC = 64;
constexpr int TILE = TR * TC;            // doubles per tile
constexpr int TILE_BYTES = TILE * 8;     // 16 KB
constexpr int ROW_GROUP = 4 * TR;        // 128 rows per forward task row group
constexpr int COL_GROUP = 4 * TC;        // 256 columns per adjoint task column group

__host__ __device__ __forceinline__ int64_t tile_offset(int64_t rb, int64_t cb, int64_t ncb) {
  return (rb * ncb + cb) * TILE;
}
__host__ __device__ __forceinline__ int col_swz(int j) { return (j >> 1) & 15; }
// position (in doubles) of element (i, j) inside its tile
__host__ __device__ __forceinline__ int in_tile(int i, int j) { return j * 32 + (i ^ col_swz(j)); }

// ---- exact-rounding arithmetic ----------------------------------------------------
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// Pairwise tree over N (power of two) leaves produced by leaf(i), i = base .. base+N-1.
template <int N, class F>
__device__ __forceinline__ double tree(const F& leaf, int base = 0) {
  if constexpr (N == 1) {
    return leaf(base);
  } else {
    const double a = tree<N / 2>(leaf, base);
    const double b = tree<N / 2>(leaf, base + N / 2);
    return add(a, b);
  }
}

// Binary-counter accumulator for a runtime number of leaves (< 2^L): push in index order,
// final() returns the pairwise tree value (absent leaves beyond the count).
template <int L>
struct Counter {
  double lvl[L];
  __device__ __forceinline__ Counter() {
#pragma unroll
    for (int l = 0; l < L; ++l) lvl[l] = 0.0;
  }
  // branch-free carry chain so lvl[] stays in registers
  __device__ __forceinline__ void push(double v, uint32_t idx) {
    bool open = true;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const bool bit = (idx >> l) & 1u;
      const double merged = add(lvl[l], v);
      const bool store = open && !bit;
      lvl[l] = store ? v : lvl[l];
      v = (open && bit) ? merged : v;
      open = open && bit;
    }
  }
  // a whole aligned subtree of 2^S leaves whose first leaf is idx << S (same carries as its
  // leaves pushed one by one)
  template <int S>
  __device__ __forceinline__ void push_node(double v, uint32_t idx) {
    bool open = true;
#pragma unroll
    for (int l = S; l < L; ++l) {
      const bool bit = (idx >> (l - S)) & 1u;
      const double merged = add(lvl[l], v);
      const bool store = open && !bit;
      lvl[l] = store ? v : lvl[l];
      v = (open && bit) ? merged : v;
      open = open && bit;
    }
  }
  __device__ __forceinline__ double final_value(uint32_t count) const {
    double acc = 0.0;
    bool have = false;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      if ((count >> l) & 1u) {
        acc = have ? add(lvl[l], acc) : lvl[l];
        have = true;
      }
    }
    return acc;
  }
};

// Butterfly over a warp: lane l holds the value of leaf block l (consecutive blocks in
// lane order); after xor-shuffles 1,2,4,8,16 every lane holds the pairwise tree value of
// the 32 blocks (IEEE addition is commutative, so both partners compute the same bits).
__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pairwise tree over a power-of-two number of values in shared memory (in place, uses
// the first n entries); all threads of the block must call it.  Returns the root.
__device__ __forceinline__ double smem_tree(double* buf, int n) {
  for (int h = n >> 1; h >= 1; h >>= 1) {
    __syncthreads();
    for (int t = threadIdx.x; t < h; t += blockDim.x) buf[t] = add(buf[2 * t], buf[2 * t + 1]);
  }
  __syncthreads();
  const double r = buf[0];
  __syncthreads();
  return r;
}

// ---- PTX wrappers: mbarrier + bulk async copy (TMA engine, UBLKCP) --------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the same wait with cluster-scope acquire: data that st.async from other CTAs completed on
// this mbarrier is visible after it returns
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(addr), "r"(rank));
  return o;
}
// 8-byte remote store into another CTA's shared memory, completing on its mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
               "d"(v), "r"(rbar)
               : "memory");
}
// global -> shared bulk copy completing on an mbarrier (bytes: multiple of 16, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// Programmatic dependent launch: wait for the preceding grid (and its memory), then let the
// next grid's CTAs be scheduled as soon as every CTA of this one is running.  Both are
// no-ops for a launch without the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_wait_and_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// launch with programmatic stream serialization (see pdl_wait_and_trigger)
template <class Kern, class... Args>
inline cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              const Args&... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a...);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One-time setup per device (kernel attributes belong to the current device's context): `f`
// runs the first time this call site is reached on each device, under a lock, so a second
// device or a second thread never launches before its attributes are set.
template <class F>
inline void once_per_device(std::atomic<unsigned long long>& done, F&& f) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}

}  // namespace l1g

// Debug timeline (L1G_TIMELINE builds only; tools/prof_solve.py --timeline): per iteration k
// and kernel, the earliest CTA entry and the earliest return from griddepcontrol.wait, by
// atomicMin of %globaltimer into a table of the kernel's translation unit.
#ifdef L1G_TIMELINE
#define L1G_TL_ENTRY const unsigned long long tl_entry__ = ::l1g::globaltimer();
#define L1G_TL_WAITED(cond, tab, kid, k)                                                 \
  if ((cond) && threadIdx.x == 0) {                                                      \
    atomicMin(&(tab)[((k) & 255) * 16 + 2 * (kid)], tl_entry__);                         \
    atomicMin(&(tab)[((k) & 255) * 16 + 2 * (kid) + 1],                                  \
              (unsigned long long)::l1g::globaltimer());                                 \
  }
#define L1G_TL_STAMP(cond, tab, slot, k) \
  if (cond) (tab)[((k) & 255) * 16 + (slot)] = (unsigned long long)::l1g::globaltimer();
#else
#define L1G_TL_ENTRY
#define L1G_TL_WAITED(cond, tab, kid, k)
#define L1G_TL_STAMP(cond, tab, slot, k)
#endif

#define L1G_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess) throw ::l1g::CudaError(e__, #call, __FILE__, __LINE__);     \
  } while (0)
