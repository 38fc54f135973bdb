// dmma.cu -- batched-RHS products on the FP64 tensor cores (BASELINE config C5).
//
// With B problems sharing one K (an isochrone campaign / regularisation path: many y or rho,
// isochrone.cpp:111-196) the per-problem GEMVs of gp_iterate (gpss.cpp:194, :211) become
//   forward  Y = K D      (n x B),  D = [d_1 .. d_B]
//   adjoint  G = K^T R'   (p x B),  R' = [r_1 + l_1 kd_1 .. ]
// i.e. two DGEMMs with 4 n p B flop per iteration, issued as mma.sync.m8n8k4.f64 (SASS
// DMMA; tcgen05 has no fp64 kind).  K stays in the tiled layout of the single-RHS kernels;
// each CTA computes a 64 x 128 (rows or columns x problems) block over one split of the
// reduction dimension, staged through shared memory with cp.async (2-3 stages); the split
// partials are joined by the finish kernels (gemv.cu), which also run every problem's
// epilogue.  DMMA accumulates with fused multiply-adds in its own order, so the batched
// path matches the per-problem canonical solve to rounding, not bit for bit.
//
// Kernels, oldest first: bfwd/badj_kernel (8 warps), b*_wide_kernel (16 warps, consumer-issued
// copies), b*_ws_kernel (16 consumer warps + a producer warp, persistent; the default).  The
// default products run on the live problems only (bcompact_kernel lists them each iteration):
// b*_ws_kernel is two instances behind one entry -- every problem in place, or the compacted
// columns with dead problem blocks / warp groups / tiles skipped -- and bws_tail_kernel takes
// the launches with at most 32 live problems (two CTAs per SM).  A column's sums do not depend
// on its place in a tile, so all of these give a problem the same bits.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "engine.h"
#include "steps.cuh"

namespace l1g {

namespace {
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp16s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace

constexpr int BW = 128;   // problems per CTA (B is padded to a multiple)
constexpr int BT = 256;   // 8 warps: 2 (rows / columns) x 4 (problems), 32 x 32 each
constexpr int VPAD = 4;   // row padding (doubles) of staged problem vectors

// K tiles are restaged column-major with a 36-double column pitch: element (i, j) of a
// tile sits at j*KP + (i ^ (col_swz(j) & 1)).  The 16-byte cp.async chunks of the global
// column runs (two adjacent rows) land whole, and both fragment patterns -- 8 rows x 4
// columns (forward) and 8 columns x 4 rows (adjoint) -- touch every 8-byte bank pair at
// most twice (KP = 36 = 4 mod 16), the minimum for 32 64-bit lanes.
constexpr int KP = 36;
constexpr int KT_S = TC * KP;  // doubles per restaged tile
__device__ __forceinline__ int kpos(int i, int j) { return j * KP + (i ^ (col_swz(j) & 1)); }
// 16-byte chunk q (0..1023) of a tile: global offset 2q, restaged offset
__device__ __forceinline__ int kchunk_dst(int q) {
  const int j = q >> 4, k2 = (q & 15) * 2;
  return j * KP + (k2 ^ (col_swz(j) & ~1));
}

// forward: K rows 64 (two tiles) x 64 columns, D chunk 128 problems x 64 columns
constexpr int F_KT = 2 * KT_S;
constexpr int F_VS = BW * (TC + VPAD);
constexpr int F_STAGE = F_KT + F_VS;
constexpr int F_STAGES = 2;
// adjoint: two tiles 64 rows x 64 columns, R chunk 128 problems x 64 rows
constexpr int A_RB = 2;  // row blocks per stage
constexpr int A_KT = A_RB * KT_S;
constexpr int A_VS = BW * (A_RB * TR + VPAD);
constexpr int A_STAGE = A_KT + A_VS;
constexpr int A_STAGES = 2;

size_t bfwd_smem() { return (size_t)F_STAGES * F_STAGE * 8; }
size_t badj_smem() { return (size_t)A_STAGES * A_STAGE * 8; }

// part[split][b][row] = sum over this split's column blocks of K[row, cols] d_b[cols]
__global__ void __launch_bounds__(BT, 1) bfwd_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wr = warp & 1, wc = warp >> 1;
  const int64_t rb0 = 2LL * blockIdx.x;
  const int split = blockIdx.y;
  const int b0 = blockIdx.z * BW;
  const int c_begin = split * a.per_split;
  const int c_end = c_begin + a.per_split < a.nblocks ? c_begin + a.per_split : a.nblocks;
  const int nch = c_end > c_begin ? c_end - c_begin : 0;
  auto load = [&](int c, int st) {
    double* ks = sm + st * F_STAGE;
    double* vs = ks + F_KT;
    const int64_t cb = c_begin + c;
    for (int q = tid; q < TILE; q += BT) {  // two tiles = 2 x 1024 chunks of 16 bytes
      const int tile = q >> 10, c = q & 1023;
      cp16(ks + tile * KT_S + kchunk_dst(c), a.K + tile_offset(rb0 + tile, cb, a.ncb) + 2 * c);
    }
    for (int q = tid; q < BW * (TC / 2); q += BT) {
      const int b = q >> 5, kq = (q & 31) * 2;
      cp16(vs + b * (TC + VPAD) + kq, a.V + (int64_t)(b0 + b) * a.vstride + cb * TC + kq);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nch > 0) load(0, 0);
  cp_commit();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) load(c + 1, (c + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* ks = sm + (c & 1) * F_STAGE + wr * KT_S;
    const double* vs = sm + (c & 1) * F_STAGE + F_KT + (wc * 32) * (TC + VPAD);
#pragma unroll 4
    for (int kk = 0; kk < TC; kk += 4) {
      const int col = kk + t;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = ks[kpos(mt * 8 + g, col)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * (TC + VPAD) + col];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
    __syncthreads();
  }
  double* out = a.part + split * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t row = (rb0 + wr) * TR + mt * 8 + g;
      const int64_t b = b0 + wc * 32 + nt * 8 + 2 * t;
      out[b * a.ostride + row] = acc[mt][nt][0];
      out[(b + 1) * a.ostride + row] = acc[mt][nt][1];
    }
}

// part[split][b][col] = sum over this split's row blocks of K[rows, col] r_b[rows]
__global__ void __launch_bounds__(BT, 1) badj_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wc = warp >> 1;
  const int64_t cb = blockIdx.x;
  const int split = blockIdx.y;
  const int b0 = blockIdx.z * BW;
  constexpr int RS = A_RB * TR + VPAD;  // row pitch of the staged R chunk
  const int r_begin = split * a.per_split;  // in row blocks (per_split is a multiple of A_RB)
  const int r_end = r_begin + a.per_split < a.nblocks ? r_begin + a.per_split : a.nblocks;
  const int nch = r_end > r_begin ? (r_end - r_begin + A_RB - 1) / A_RB : 0;
  auto load = [&](int c, int st) {
    double* ks = sm + st * A_STAGE;
    double* vs = ks + A_KT;
    const int64_t rb = r_begin + (int64_t)c * A_RB;
    for (int q = tid; q < A_RB * TILE / 2; q += BT) {
      const int tl = q >> 10, cq = q & 1023;
      cp16(ks + tl * KT_S + kchunk_dst(cq), a.K + tile_offset(rb + tl, cb, a.ncb) + 2 * cq);
    }
    for (int q = tid; q < BW * (A_RB * TR / 2); q += BT) {
      const int b = q >> 5, kq = (q & 31) * 2;
      cp16(vs + b * RS + kq, a.V + (int64_t)(b0 + b) * a.vstride + rb * TR + kq);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nch > 0) load(0, 0);
  cp_commit();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) load(c + 1, (c + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* ks = sm + (c & 1) * A_STAGE;
    const double* vs = sm + (c & 1) * A_STAGE + A_KT + (wc * 32) * RS;
#pragma unroll 4
    for (int kk = 0; kk < A_RB * TR; kk += 4) {
      const int row = kk + t;
      const double* kt = ks + (row >> 5) * KT_S;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = kt[kpos(row & 31, wm * 32 + mt * 8 + g)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * RS + row];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
    __syncthreads();
  }
  double* out = a.part + split * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t col = cb * TC + wm * 32 + mt * 8 + g;
      const int64_t b = b0 + wc * 32 + nt * 8 + 2 * t;
      out[b * a.ostride + col] = acc[mt][nt][0];
      out[(b + 1) * a.ostride + col] = acc[mt][nt][1];
    }
}

// ---------------------------------------------------------------- 16-warp products
// CTA tile 128 (rows | columns) x 128 problems, 16 warps of 32 x 32, k-chunks of 32 and a
// 3-stage cp.async ring (73.7 KB per stage): twice the warps per SM of the 8-warp kernels
// above, each staged K element reused by 128 problems and each staged vector by 128 outputs.
constexpr int WT = 512;             // threads
constexpr int W_KS = 4 * TR * KP;   // restaged K per stage: 4 x (32 columns x KP)
constexpr int W_VP = 32 + VPAD;     // pitch of a staged 32-long vector chunk
constexpr int W_VS = BW * W_VP;
constexpr int W_STAGE = W_KS + W_VS;
constexpr int W_STAGES = 3;
size_t bwide_smem() { return (size_t)W_STAGES * W_STAGE * 8; }

// forward: part[split][b][row] over this split's 32-column chunks (per_split chunks each)
__global__ void __launch_bounds__(WT, 1) bfwd_wide_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wr = warp & 3, wc = warp >> 2;
  const int64_t rb0 = 4LL * blockIdx.x;
  const int b0 = blockIdx.z * BW;
  const int nchunk = 2 * a.nblocks;  // 32-column chunks
  const int c_begin = blockIdx.y * a.per_split;
  const int c_end = c_begin + a.per_split < nchunk ? c_begin + a.per_split : nchunk;
  const int nch = c_end > c_begin ? c_end - c_begin : 0;
  // per-thread copy offsets, fixed across chunks: K chunk tid of 4 row blocks (the 16-byte
  // chunks of half a tile), V rows tid/16 + 32 i at column pair tid%16
  const uint32_t s_base = smem_u32(sm);
  const uint32_t s_k = (uint32_t)kchunk_dst(tid) * 8u;
  const uint32_t s_v = (uint32_t)(W_KS + (tid >> 4) * W_VP + (tid & 15) * 2) * 8u;
  const double* g_k = a.K + rb0 * a.ncb * TILE + 2 * tid;
  const int64_t k_rs = a.ncb * TILE;  // one row block further
  const double* g_v = a.V + (int64_t)(b0 + (tid >> 4)) * a.vstride + (tid & 15) * 2;
  const int64_t v_rs = 32 * a.vstride;
  auto load = [&](int c, int st) {
    const int64_t ch = c_begin + c, cb = ch >> 1, half = ch & 1;
    const uint32_t so = s_base + (uint32_t)(st * W_STAGE) * 8u;
    const double* gk = g_k + cb * TILE + half * (TILE / 2);
#pragma unroll
    for (int r = 0; r < 4; ++r) cp16s(so + s_k + (uint32_t)(r * TR * KP * 8), gk + r * k_rs);
    const double* gv = g_v + ch * 32;
#pragma unroll
    for (int i = 0; i < 4; ++i) cp16s(so + s_v + (uint32_t)(i * 32 * W_VP * 8), gv + i * v_rs);
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int st = 0; st < W_STAGES - 1; ++st) {
    if (st < nch) load(st, st);
    cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_wait<W_STAGES - 2>();
    __syncthreads();  // chunk c landed; the stage of chunk c - 1 is free
    if (c + W_STAGES - 1 < nch) load(c + W_STAGES - 1, (c + W_STAGES - 1) % W_STAGES);
    cp_commit();
    const double* ks = sm + (c % W_STAGES) * W_STAGE + wr * (TR * KP);
    const double* vs = sm + (c % W_STAGES) * W_STAGE + W_KS + (wc * 32) * W_VP;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const int col = kk + t;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = ks[kpos(mt * 8 + g, col)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * W_VP + col];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
  }
  double* out = a.part + blockIdx.y * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t row = (rb0 + wr) * TR + mt * 8 + g;
      const int64_t b = b0 + wc * 32 + nt * 8 + 2 * t;
      out[b * a.ostride + row] = acc[mt][nt][0];
      out[(b + 1) * a.ostride + row] = acc[mt][nt][1];
    }
}

// adjoint: part[split][b][col] over this split's row blocks (per_split each); a CTA covers
// two column blocks (128 columns)
__global__ void __launch_bounds__(WT, 1) badj_wide_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wc = warp >> 2;
  const int64_t cb0 = 2LL * blockIdx.x;
  const int b0 = blockIdx.z * BW;
  const int r_begin = blockIdx.y * a.per_split;
  const int r_end = r_begin + a.per_split < a.nblocks ? r_begin + a.per_split : a.nblocks;
  const int nch = r_end > r_begin ? r_end - r_begin : 0;
  // per-thread copy offsets, fixed across chunks: 16-byte chunks tid and tid + 512 of the two
  // tiles (chunk j + 32 columns has the same swizzle: offset + 32 KP), V rows tid/16 + 32 i
  const uint32_t s_base = smem_u32(sm);
  const uint32_t s_k = (uint32_t)kchunk_dst(tid) * 8u;
  const uint32_t s_v = (uint32_t)(W_KS + (tid >> 4) * W_VP + (tid & 15) * 2) * 8u;
  const double* g_k = a.K + cb0 * TILE + 2 * tid;
  const double* g_v = a.V + (int64_t)(b0 + (tid >> 4)) * a.vstride + (tid & 15) * 2;
  const int64_t v_rs = 32 * a.vstride;
  auto load = [&](int c, int st) {
    const int64_t rb = r_begin + c;
    const uint32_t so = s_base + (uint32_t)(st * W_STAGE) * 8u;
    const double* gk = g_k + rb * a.ncb * TILE;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      cp16s(so + s_k + (uint32_t)(((i >> 1) * KT_S + (i & 1) * 32 * KP) * 8),
            gk + (i >> 1) * TILE + (i & 1) * 1024);
    const double* gv = g_v + rb * TR;
#pragma unroll
    for (int i = 0; i < 4; ++i) cp16s(so + s_v + (uint32_t)(i * 32 * W_VP * 8), gv + i * v_rs);
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int st = 0; st < W_STAGES - 1; ++st) {
    if (st < nch) load(st, st);
    cp_commit();
  }
  const int tl = wm >> 1, cofs = (wm & 1) * 32;
  for (int c = 0; c < nch; ++c) {
    cp_wait<W_STAGES - 2>();
    __syncthreads();
    if (c + W_STAGES - 1 < nch) load(c + W_STAGES - 1, (c + W_STAGES - 1) % W_STAGES);
    cp_commit();
    const double* kt = sm + (c % W_STAGES) * W_STAGE + tl * KT_S;
    const double* vs = sm + (c % W_STAGES) * W_STAGE + W_KS + (wc * 32) * W_VP;
#pragma unroll
    for (int kk = 0; kk < TR; kk += 4) {
      const int row = kk + t;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = kt[kpos(row, cofs + mt * 8 + g)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * W_VP + row];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
  }
  double* out = a.part + blockIdx.y * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t col = (cb0 + tl) * TC + cofs + mt * 8 + g;
      const int64_t b = b0 + wc * 32 + nt * 8 + 2 * t;
      out[b * a.ostride + col] = acc[mt][nt][0];
      out[(b + 1) * a.ostride + col] = acc[mt][nt][1];
    }
}

// ---------------------------------------------------------------- producer-warp products
// The 16-warp products with the copies taken off the consumers: a 17th warp issues every
// cp.async of a stage (the 512 consumer threads' share, 128 copies per lane) and its lanes'
// cp.async arrivals complete the stage's `full` mbarrier; each consumer warp waits only for
// the stage it reads and marks it `empty` when done, so consumers never wait for each other
// and the DMMA pipe is not drained at every chunk boundary.
constexpr int WP = WT + 32;  // 16 consumer warps + 1 producer warp
#ifndef L1G_TAIL_NT
#define L1G_TAIL_NT 4
#endif
constexpr int T_MAXNT = L1G_TAIL_NT;      // 8-problem tiles the few-live-problems variant takes
constexpr int T_VROWS = 8 * T_MAXNT;      // i.e. live problems (bws_tail_kernel)
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Persistent: CTA i takes work items i, i + grid, ... (item = (row tile, split, problem
// block) in the order of the former grid), and the ring runs on across items, so the next
// item's first stages load while the consumers finish the current one.
struct WsItem {
  int x, y, z;
};
// Live-problem compaction (BGemmArgs::active / nact): the product's column j of problem
// block b0 is problem active[b0 + j]; columns past the live count are not computed.
__device__ __forceinline__ int ws_live(int na, int b0) {
  const int nl = na - b0;
  return nl < 0 ? 0 : (nl > BW ? BW : nl);
}
__device__ __forceinline__ int ws_tiles(int nl, int wc) {  // live 8-problem tiles of group wc
  const int wl = nl - wc * 32;
  return wl <= 0 ? 0 : (wl >= 32 ? 4 : (wl + 7) >> 3);
}
__device__ __forceinline__ int64_t ws_problem(const int* active, int b0, int j) {
  return active ? (int64_t)__ldg(active + b0 + j) : (int64_t)(b0 + j);
}
// the producer warp's table of source rows (columns past the live count repeat the last one,
// so a partly live tile reads valid memory)
// Returns true when the block is whole and in place (column j is problem b0 + j): the copies
// then use plain strides instead of the table.
__device__ __forceinline__ bool ws_fill_rows(int* s_act, const int* active, int b0, int nl, int lane) {
  __syncwarp();
  bool same = nl == BW;
  for (int j = lane; j < BW; j += 32) {
    const int jj = j < nl ? j : nl - 1;
    const int b = active ? __ldg(active + b0 + jj) : b0 + jj;
    s_act[j] = b;
    same &= b == b0 + j;
  }
  __syncwarp();
  return __all_sync(0xffffffffu, same);
}
__device__ __forceinline__ WsItem ws_item(int it, int nx, int ny) {
  WsItem w;
  w.x = it % nx;
  w.y = (it / nx) % ny;
  w.z = it / (nx * ny);
  return w;
}

// CP = false: every problem live and in place (the code without any of the compaction);
// CP = true: columns gathered through active[], dead blocks / groups / tiles skipped.
template <bool CP>
__device__ __forceinline__ void bfwd_ws_impl(const BGemmArgs& a, const int na) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t full[W_STAGES], empty[W_STAGES];
  __shared__ int s_act[CP ? BW : 1];  // producer warp only
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int nchunk = 2 * a.nblocks;  // 32-column chunks
  const int nitems = a.nx * a.ny * a.nz;
  auto nch_of = [&](const WsItem& w) {
    const int c_begin = w.y * a.per_split;
    const int c_end = c_begin + a.per_split < nchunk ? c_begin + a.per_split : nchunk;
    return c_end > c_begin ? c_end - c_begin : 0;
  };
  if (tid == 0) {
    for (int st = 0; st < W_STAGES; ++st) {
      mbar_init(&full[st], 32);
      mbar_init(&empty[st], WT / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == WT / 32) {  // ---- producer: the copies of all 512 consumer threads
    const uint32_t s_base = smem_u32(sm);
    const int64_t k_rs = a.ncb * TILE;
    const int64_t v_rs = 32 * a.vstride;
    int gc = 0;  // ring position across items
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
     const WsItem w = ws_item(it, a.nx, a.ny);
     const int64_t rb0 = 4LL * w.x;
     const int b0 = w.z * BW;
     const int nl = CP ? ws_live(na, b0) : BW;
     if (CP && nl == 0) continue;  // no live problem in this block (the consumers skip it too)
     const bool inplace = CP ? ws_fill_rows(s_act, a.active, b0, nl, lane) : true;
     const int nl8 = (nl + 7) & ~7;
     const int c_begin = w.y * a.per_split, nch = nch_of(w);
     for (int c = 0; c < nch; ++c, ++gc) {
      const int st = gc % W_STAGES;
      if (gc >= W_STAGES) mbar_wait(&empty[st], (uint32_t)((gc / W_STAGES - 1) & 1));
      const int64_t ch = c_begin + c, cb = ch >> 1, half = ch & 1;
      const uint32_t so = s_base + (uint32_t)(st * W_STAGE) * 8u;
      const double* gk = a.K + rb0 * k_rs + cb * TILE + half * (TILE / 2);
      const double* gv = a.V + ch * 32;
      if (!CP || inplace) {
        const double* gvb = gv + (int64_t)b0 * a.vstride;
#pragma unroll 4
        for (int vt = lane; vt < WT; vt += 32) {
          const uint32_t s_k = so + (uint32_t)kchunk_dst(vt) * 8u;
          const double* k0 = gk + 2 * vt;
#pragma unroll
          for (int r = 0; r < 4; ++r) cp16s(s_k + (uint32_t)(r * TR * KP * 8), k0 + r * k_rs);
          const uint32_t s_v = so + (uint32_t)(W_KS + (vt >> 4) * W_VP + (vt & 15) * 2) * 8u;
          const double* v0 = gvb + (int64_t)(vt >> 4) * a.vstride + (vt & 15) * 2;
#pragma unroll
          for (int i = 0; i < 4; ++i) cp16s(s_v + (uint32_t)(i * 32 * W_VP * 8), v0 + i * v_rs);
        }
      } else {
#pragma unroll 4
        for (int vt = lane; vt < WT; vt += 32) {
          const uint32_t s_k = so + (uint32_t)kchunk_dst(vt) * 8u;
          const double* k0 = gk + 2 * vt;
#pragma unroll
          for (int r = 0; r < 4; ++r) cp16s(s_k + (uint32_t)(r * TR * KP * 8), k0 + r * k_rs);
        }
        // the live columns' vector chunks only (16 copies of 16 bytes per column; tiles past
        // nl8 are never read)
#pragma unroll 2
        for (int idx = lane; idx < nl8 * 16; idx += 32) {
          const int j = idx >> 4, cc = (idx & 15) * 2;
          cp16s(so + (uint32_t)(W_KS + j * W_VP + cc) * 8u, gv + (int64_t)s_act[j] * a.vstride + cc);
        }
      }
      cp_arrive_noinc(&full[st]);
     }
    }
    cp_wait<0>();
    return;
  }
  // ---- consumers
  const int wr = warp & 3, wc = warp >> 2;
  int gc = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
  const WsItem w = ws_item(it, a.nx, a.ny);
  const int64_t rb0 = 4LL * w.x;
  const int b0 = w.z * BW;
  const int nl = CP ? ws_live(na, b0) : BW;
  if (CP && nl == 0) continue;
  const int ntl = CP ? ws_tiles(nl, wc) : 4;  // live 8-problem tiles of this warp's 32-problem group
  const int nch = nch_of(w);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (!CP || ntl == 4) {  // a whole group: the full 32 x 32 warp tile
  for (int c = 0; c < nch; ++c, ++gc) {
    const int st = gc % W_STAGES;
    mbar_wait(&full[st], (uint32_t)((gc / W_STAGES) & 1));
    const double* ks = sm + st * W_STAGE + wr * (TR * KP);
    const double* vs = sm + st * W_STAGE + W_KS + (wc * 32) * W_VP;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const int col = kk + t;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = ks[kpos(mt * 8 + g, col)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * W_VP + col];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  } else {  // a partly live group: only its live tiles (same sums per problem); a dead one
            // just keeps the ring's barriers in step
  for (int c = 0; c < nch; ++c, ++gc) {
    const int st = gc % W_STAGES;
    mbar_wait(&full[st], (uint32_t)((gc / W_STAGES) & 1));
    const double* ks = sm + st * W_STAGE + wr * (TR * KP);
    const double* vs = sm + st * W_STAGE + W_KS + (wc * 32) * W_VP;
    if (ntl > 0) {
#pragma unroll 2
      for (int kk = 0; kk < 32; kk += 4) {
        const int col = kk + t;
        double av[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) av[mt] = ks[kpos(mt * 8 + g, col)];
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
          if (nt < ntl) {
            const double bv = vs[(nt * 8 + g) * W_VP + col];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) dmma884(acc[mt][nt], av[mt], bv);
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  }
  double* out = a.part + w.y * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t row = (rb0 + wr) * TR + mt * 8 + g;
      const int j = wc * 32 + nt * 8 + 2 * t;  // column of the product
      if (!CP) {
        out[(int64_t)(b0 + j) * a.ostride + row] = acc[mt][nt][0];
        out[(int64_t)(b0 + j + 1) * a.ostride + row] = acc[mt][nt][1];
      } else {
        if (j < nl) out[ws_problem(a.active, b0, j) * a.ostride + row] = acc[mt][nt][0];
        if (j + 1 < nl) out[ws_problem(a.active, b0, j + 1) * a.ostride + row] = acc[mt][nt][1];
      }
    }
  }
}

// (its own function: the all-live path above keeps its registers and schedule)
__device__ __noinline__ void bfwd_ws_compact(const BGemmArgs& a, const int na) { bfwd_ws_impl<true>(a, na); }

__global__ void __launch_bounds__(WP, 1) bfwd_ws_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  const int na = a.nact ? __ldcg(a.nact) : a.nz * BW;  // live problems (compacted columns)
  if (a.tail && na <= T_VROWS) return;               // bws_tail_kernel takes this launch
  // all live -- or so many that no 32-problem group could be skipped: every problem in place
  // (the gather costs more than the few dead columns; stopped problems' columns are ignored)
  if ((na + 31) / 32 >= (a.nb + 31) / 32) bfwd_ws_impl<false>(a, na);
  else bfwd_ws_compact(a, na);
}

template <bool CP>
__device__ __forceinline__ void badj_ws_impl(const BGemmArgs& a, const int na) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t full[W_STAGES], empty[W_STAGES];
  __shared__ int s_act[CP ? BW : 1];  // producer warp only
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int nitems = a.nx * a.ny * a.nz;
  auto nch_of = [&](const WsItem& w) {
    const int r_begin = w.y * a.per_split;
    const int r_end = r_begin + a.per_split < a.nblocks ? r_begin + a.per_split : a.nblocks;
    return r_end > r_begin ? r_end - r_begin : 0;
  };
  if (tid == 0) {
    for (int st = 0; st < W_STAGES; ++st) {
      mbar_init(&full[st], 32);
      mbar_init(&empty[st], WT / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == WT / 32) {  // ---- producer
    const uint32_t s_base = smem_u32(sm);
    const int64_t v_rs = 32 * a.vstride;
    int gc = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
     const WsItem w = ws_item(it, a.nx, a.ny);
     const int64_t cb0 = 2LL * w.x;
     const int b0 = w.z * BW;
     const int nl = CP ? ws_live(na, b0) : BW;
     if (CP && nl == 0) continue;
     const bool inplace = CP ? ws_fill_rows(s_act, a.active, b0, nl, lane) : true;
     const int nl8 = (nl + 7) & ~7;
     const int r_begin = w.y * a.per_split, nch = nch_of(w);
     for (int c = 0; c < nch; ++c, ++gc) {
      const int st = gc % W_STAGES;
      if (gc >= W_STAGES) mbar_wait(&empty[st], (uint32_t)((gc / W_STAGES - 1) & 1));
      const int64_t rb = r_begin + c;
      const uint32_t so = s_base + (uint32_t)(st * W_STAGE) * 8u;
      const double* gk = a.K + (rb * a.ncb + cb0) * TILE;
      const double* gv = a.V + rb * TR;
      if (!CP || inplace) {
        const double* gvb = gv + (int64_t)b0 * a.vstride;
#pragma unroll 4
        for (int vt = lane; vt < WT; vt += 32) {
          const uint32_t s_k = so + (uint32_t)kchunk_dst(vt) * 8u;
          const double* k0 = gk + 2 * vt;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            cp16s(s_k + (uint32_t)(((i >> 1) * KT_S + (i & 1) * 32 * KP) * 8),
                  k0 + (i >> 1) * TILE + (i & 1) * 1024);
          const uint32_t s_v = so + (uint32_t)(W_KS + (vt >> 4) * W_VP + (vt & 15) * 2) * 8u;
          const double* v0 = gvb + (int64_t)(vt >> 4) * a.vstride + (vt & 15) * 2;
#pragma unroll
          for (int i = 0; i < 4; ++i) cp16s(s_v + (uint32_t)(i * 32 * W_VP * 8), v0 + i * v_rs);
        }
      } else {
#pragma unroll 4
        for (int vt = lane; vt < WT; vt += 32) {
          const uint32_t s_k = so + (uint32_t)kchunk_dst(vt) * 8u;
          const double* k0 = gk + 2 * vt;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            cp16s(s_k + (uint32_t)(((i >> 1) * KT_S + (i & 1) * 32 * KP) * 8),
                  k0 + (i >> 1) * TILE + (i & 1) * 1024);
        }
#pragma unroll 2
        for (int idx = lane; idx < nl8 * 16; idx += 32) {
          const int j = idx >> 4, cc = (idx & 15) * 2;
          cp16s(so + (uint32_t)(W_KS + j * W_VP + cc) * 8u, gv + (int64_t)s_act[j] * a.vstride + cc);
        }
      }
      cp_arrive_noinc(&full[st]);
     }
    }
    cp_wait<0>();
    return;
  }
  // ---- consumers
  const int wm = warp & 3, wc = warp >> 2;
  const int tl = wm >> 1, cofs = (wm & 1) * 32;
  int gc = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
  const WsItem w = ws_item(it, a.nx, a.ny);
  const int64_t cb0 = 2LL * w.x;
  const int b0 = w.z * BW;
  const int nl = CP ? ws_live(na, b0) : BW;
  if (CP && nl == 0) continue;
  const int ntl = CP ? ws_tiles(nl, wc) : 4;
  const int nch = nch_of(w);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (!CP || ntl == 4) {
  for (int c = 0; c < nch; ++c, ++gc) {
    const int st = gc % W_STAGES;
    mbar_wait(&full[st], (uint32_t)((gc / W_STAGES) & 1));
    const double* kt = sm + st * W_STAGE + tl * KT_S;
    const double* vs = sm + st * W_STAGE + W_KS + (wc * 32) * W_VP;
#pragma unroll
    for (int kk = 0; kk < TR; kk += 4) {
      const int row = kk + t;
      double av[4], bv[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = kt[kpos(row, cofs + mt * 8 + g)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bv[nt] = vs[(nt * 8 + g) * W_VP + row];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  } else {
  for (int c = 0; c < nch; ++c, ++gc) {
    const int st = gc % W_STAGES;
    mbar_wait(&full[st], (uint32_t)((gc / W_STAGES) & 1));
    const double* kt = sm + st * W_STAGE + tl * KT_S;
    const double* vs = sm + st * W_STAGE + W_KS + (wc * 32) * W_VP;
    if (ntl > 0) {
#pragma unroll 2
      for (int kk = 0; kk < TR; kk += 4) {
        const int row = kk + t;
        double av[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) av[mt] = kt[kpos(row, cofs + mt * 8 + g)];
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
          if (nt < ntl) {
            const double bv = vs[(nt * 8 + g) * W_VP + row];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) dmma884(acc[mt][nt], av[mt], bv);
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  }
  double* out = a.part + w.y * a.pslab;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t col = (cb0 + tl) * TC + cofs + mt * 8 + g;
      const int j = wc * 32 + nt * 8 + 2 * t;
      if (!CP) {
        out[(int64_t)(b0 + j) * a.ostride + col] = acc[mt][nt][0];
        out[(int64_t)(b0 + j + 1) * a.ostride + col] = acc[mt][nt][1];
      } else {
        if (j < nl) out[ws_problem(a.active, b0, j) * a.ostride + col] = acc[mt][nt][0];
        if (j + 1 < nl) out[ws_problem(a.active, b0, j + 1) * a.ostride + col] = acc[mt][nt][1];
      }
    }
  }
}

// (its own function: the all-live path above keeps its registers and schedule)
__device__ __noinline__ void badj_ws_compact(const BGemmArgs& a, const int na) { badj_ws_impl<true>(a, na); }

__global__ void __launch_bounds__(WP, 1) badj_ws_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  const int na = a.nact ? __ldcg(a.nact) : a.nz * BW;
  if (a.tail && na <= T_VROWS) return;
  if ((na + 31) / 32 >= (a.nb + 31) / 32) badj_ws_impl<false>(a, na);
  else badj_ws_compact(a, na);
}

// ---------------------------------------------------------------- few live problems
// With few live problems a product is bound by one accumulator's dependent DMMA chain along the
// reduction (an item takes 128 m8n8k4 steps in a row), not by the tensor pipe or by HBM.  This
// variant runs two CTAs per SM -- four consumer warps (32 rows or columns x the live problems
// each) and a producer warp, two stages of [K tiles | live vector rows] -- so two items' chains
// run side by side on every SM.  NT = 1: at most 8 live problems (one 8-problem tile per warp);
// NT = 4: at most 32.  Same chunks in the same order per accumulator, so the bits are those of
// the full-size kernels.  Both launches sit in the iteration; the live count picks one (the other
// returns at once).
constexpr int T_CW = 4;
constexpr int T_THREADS = 32 * (T_CW + 1);
constexpr int T_STAGES = 2;
constexpr int T_MAXROWS = 8 * T_MAXNT;
size_t btail_smem() { return (size_t)T_STAGES * (W_KS + 8 * T_MAXNT * W_VP) * 8; }  // [K | rows] x 2

template <bool ADJ, int NT>
__device__ __forceinline__ void bws_tail_body(const BGemmArgs& a, const int na) {
  constexpr int VROWS = 8 * NT, STAGE = W_KS + 8 * NT * W_VP;  // doubles per stage
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t full[T_STAGES], empty[T_STAGES];
  __shared__ int s_act[VROWS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int nitems = a.nx * a.ny;  // the live problems are the leading columns of block 0
  const int nred = ADJ ? a.nblocks : 2 * a.nblocks;  // reduction chunks (row blocks | 32 columns)
  auto nch_of = [&](const WsItem& w) {
    const int c_begin = w.y * a.per_split;
    const int c_end = c_begin + a.per_split < nred ? c_begin + a.per_split : nred;
    return c_end > c_begin ? c_end - c_begin : 0;
  };
  if (tid == 0) {
    for (int st = 0; st < T_STAGES; ++st) {
      mbar_init(&full[st], 32);
      mbar_init(&empty[st], T_CW);
    }
    fence_barrier_init();
  }
  if (tid < VROWS) s_act[tid] = __ldg(a.active + (tid < na ? tid : na - 1));
  __syncthreads();
  const int nl8 = (na + 7) & ~7;  // vector rows staged (whole 8-problem tiles)
  if (warp == T_CW) {  // ---- producer
    const uint32_t s_base = smem_u32(sm);
    const int64_t k_rs = a.ncb * TILE;
    int gc = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const WsItem w = ws_item(it, a.nx, a.ny);
      const int c_begin = w.y * a.per_split, nch = nch_of(w);
      for (int c = 0; c < nch; ++c, ++gc) {
        const int st = gc % T_STAGES;
        if (gc >= T_STAGES) mbar_wait(&empty[st], (uint32_t)((gc / T_STAGES - 1) & 1));
        const uint32_t so = s_base + (uint32_t)(st * STAGE) * 8u;
        const int64_t ch = c_begin + c;
        const double* gk;
        const double* gv;
        if (ADJ) {
          gk = a.K + (ch * a.ncb + 2LL * w.x) * TILE;
          gv = a.V + ch * TR;
        } else {
          gk = a.K + 4LL * w.x * k_rs + (ch >> 1) * TILE + (ch & 1) * (TILE / 2);
          gv = a.V + ch * 32;
        }
#pragma unroll 4
        for (int vt = lane; vt < WT; vt += 32) {
          const uint32_t s_k = so + (uint32_t)kchunk_dst(vt) * 8u;
          const double* k0 = gk + 2 * vt;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (ADJ)
              cp16s(s_k + (uint32_t)(((i >> 1) * KT_S + (i & 1) * 32 * KP) * 8),
                    k0 + (i >> 1) * TILE + (i & 1) * 1024);
            else
              cp16s(s_k + (uint32_t)(i * TR * KP * 8), k0 + i * k_rs);
          }
        }
#pragma unroll 2
        for (int idx = lane; idx < nl8 * 16; idx += 32) {
          const int j = idx >> 4, cc = (idx & 15) * 2;
          cp16s(so + (uint32_t)(W_KS + j * W_VP + cc) * 8u, gv + (int64_t)s_act[j] * a.vstride + cc);
        }
        cp_arrive_noinc(&full[st]);
      }
    }
    cp_wait<0>();
    return;
  }
  // ---- consumers: warp = row block of the tile (forward) / 32-column group (adjoint)
  const int tl = warp >> 1, cofs = (warp & 1) * 32;
  const int ntl = nl8 >> 3;  // live tiles (1 .. NT)
  int gc = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const WsItem w = ws_item(it, a.nx, a.ny);
    const int nch = nch_of(w);
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    for (int c = 0; c < nch; ++c, ++gc) {
      const int st = gc % T_STAGES;
      mbar_wait(&full[st], (uint32_t)((gc / T_STAGES) & 1));
      const double* kb = sm + st * STAGE + (ADJ ? tl * KT_S : warp * (TR * KP));
      const double* vs = sm + st * STAGE + W_KS;
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        const int q = kk + t;  // column of the chunk (forward) / row of the block (adjoint)
        double av[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
          av[mt] = ADJ ? kb[kpos(q, cofs + mt * 8 + g)] : kb[kpos(mt * 8 + g, q)];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          if (NT == 1 || nt < ntl) {
            const double bv = vs[(nt * 8 + g) * W_VP + q];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) dmma884(acc[mt][nt], av[mt], bv);
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double* out = a.part + w.y * a.pslab;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int64_t o = ADJ ? (2LL * w.x + tl) * TC + cofs + mt * 8 + g
                              : (4LL * w.x + warp) * TR + mt * 8 + g;
        const int j = nt * 8 + 2 * t;
        if (j < na) out[(int64_t)s_act[j] * a.ostride + o] = acc[mt][nt][0];
        if (j + 1 < na) out[(int64_t)s_act[j + 1] * a.ostride + o] = acc[mt][nt][1];
      }
  }
}

template <bool ADJ>
__global__ void __launch_bounds__(T_THREADS, 2) bws_tail_kernel(const BGemmArgs a) {
  pdl_wait_and_trigger();
  const int na = __ldcg(a.nact);
  if (na <= 0 || na > T_MAXROWS) return;  // the full-size kernel takes this launch
  if (na <= 8) bws_tail_body<ADJ, 1>(a, na);
  else bws_tail_body<ADJ, T_MAXNT>(a, na);
}

template <int NA>
__device__ __forceinline__ void warp_tree_arrays_b(const double* v, int count, int stride,
                                                   int lane, double* out) {
  Counter<11> acc[NA];  // groups < 2^16
  const int chunks = (count + 31) >> 5;
  for (int c0 = 0; c0 < chunks; c0 += 4) {
    double x[4][NA];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = (c0 + u) * 32 + lane;
#pragma unroll
      for (int j = 0; j < NA; ++j) x[u][j] = i < count ? __ldcg(v + (int64_t)i * stride + j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < chunks)
#pragma unroll
        for (int j = 0; j < NA; ++j) acc[j].push(warp_tree(x[u][j]), (uint32_t)(c0 + u));
  }
#pragma unroll
  for (int j = 0; j < NA; ++j) out[j] = acc[j].final_value((uint32_t)chunks);
}

// ---------------------------------------------------------------- batched finishes
// One warp per (problem, 32 rows | 64 columns): the split partials are joined in split
// order by a binary counter (pairwise), then the problem's epilogue runs as in the
// single-RHS finish kernels; the problem's last warp (per-problem counter) joins the group
// values and runs the scalar tail (steps.cuh).
constexpr int BF_W = 8;  // warps (problems) per CTA

__global__ void __launch_bounds__(32 * BF_W) bfin_fwd_kernel(const BFinArgs a) {
  pdl_wait_and_trigger();
  __shared__ DevState snap[BF_W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y * BF_W + warp;
  if (b >= a.B) return;
  DevState* st = a.st ? a.st + b : nullptr;
  if (a.mode != FWD_APPLY && st->status != RUNNING) return;
  const int64_t row = (int64_t)blockIdx.x * 32 + lane;
  const int64_t ob = (int64_t)b * a.ostride;
  Counter<8> acc;  // splits < 256
  int k = 0;
  for (; k + 4 <= a.splits; k += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(a.part + (k + u) * a.pslab + ob + row);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc.push(v[u], (uint32_t)(k + u));
  }
  for (; k < a.splits; ++k) acc.push(__ldcg(a.part + k * a.pslab + ob + row), (uint32_t)k);
  const double kd = acc.final_value((uint32_t)a.splits);
  if (a.mode == FWD_APPLY) {
    a.vout[ob + row] = kd;
    return;
  }
  const int cur = st->cur;
  double l0, l1 = 0.0;
  if (a.mode == FWD_INIT) {
    const double r = sub(kd, a.vb.y[ob + row]);  // Kx0 - y   (gpss.cpp:128)
    a.vb.r[cur][ob + row] = r;
    l0 = mul(r, r);
  } else {
    a.vb.kd[ob + row] = kd;
    l0 = mul(a.vb.r[cur][ob + row], kd);           // (Kx-y)'Kd (gpss.cpp:195)
    l1 = mul(kd, kd);                              // ||Kd||^2  (gpss.cpp:196)
  }
  l0 = warp_tree(l0);
  l1 = warp_tree(l1);
  const int ngrp = gridDim.x;
  double* grp = a.grpsum + (int64_t)b * a.grp_stride;
  unsigned last = 0;
  if (lane == 0) {
    grp[2 * blockIdx.x + 0] = l0;
    grp[2 * blockIdx.x + 1] = l1;
    __threadfence();
    last = atomicAdd(a.counters + b, 1u) == (unsigned)ngrp - 1u;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  double AB[2];
  warp_tree_arrays_b<2>(grp, ngrp, 2, lane, AB);
  snapshot(&snap[warp], st, lane);
  if (lane != 0) return;
  a.counters[b] = 0;
  fwd_tail(st, snap[warp], a.mode, AB[0], AB[1]);
}

__global__ void __launch_bounds__(32 * BF_W) bfin_adj_kernel(const BFinArgs a) {
  pdl_wait_and_trigger();
  __shared__ DevState snap[BF_W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y * BF_W + warp;
  if (b >= a.B) return;
  DevState* st = a.st ? a.st + b : nullptr;
  if (a.mode != ADJ_APPLY && st->status != RUNNING) return;
  const int64_t col = (int64_t)blockIdx.x * 64 + 2 * lane;
  const int64_t ob = (int64_t)b * a.ostride;
  Counter<8> acc0, acc1;
  int k = 0;
  for (; k + 4 <= a.splits; k += 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = __ldcg(reinterpret_cast<const double2*>(a.part + (k + u) * a.pslab + ob + col));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc0.push(v[u].x, (uint32_t)(k + u));
      acc1.push(v[u].y, (uint32_t)(k + u));
    }
  }
  for (; k < a.splits; ++k) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(a.part + k * a.pslab + ob + col));
    acc0.push(v.x, (uint32_t)k);
    acc1.push(v.y, (uint32_t)k);
  }
  const double s0 = acc0.final_value((uint32_t)a.splits), s1 = acc1.final_value((uint32_t)a.splits);
  if (a.mode == ADJ_APPLY) {
    *reinterpret_cast<double2*>(a.vout + ob + col) = make_double2(s0, s1);
    return;
  }
  const int cur = st->cur;
  const double g0 = mul(2.0, s0), g1 = mul(2.0, s1);  // 2 K^T r (gpss.cpp:130, :211)
  if (a.mode == ADJ_INIT) {
    *reinterpret_cast<double2*>(a.vb.g[cur] + ob + col) = make_double2(g0, g1);
    return;
  }
  const double lam = st->step;
  const double2 xo = *reinterpret_cast<const double2*>(a.vb.x[cur] + ob + col);
  const double2 go = *reinterpret_cast<const double2*>(a.vb.g[cur] + ob + col);
  const double2 dd = *reinterpret_cast<const double2*>(a.vb.d + ob + col);
  const double x0n = add(xo.x, mul(lam, dd.x)), x1n = add(xo.y, mul(lam, dd.y));
  *reinterpret_cast<double2*>(a.vb.x[cur ^ 1] + ob + col) = make_double2(x0n, x1n);
  *reinterpret_cast<double2*>(a.vb.g[cur ^ 1] + ob + col) = make_double2(g0, g1);
  const double sa = sub(x0n, xo.x), sb = sub(x1n, xo.y);
  const double za = sub(g0, go.x), zb = sub(g1, go.y);
  const double dsz = warp_tree(add(mul(sa, za), mul(sb, zb)));
  const double dss = warp_tree(add(mul(sa, sa), mul(sb, sb)));
  const double dzz = warp_tree(add(mul(za, za), mul(zb, zb)));
  const int ngrp = gridDim.x;
  double* grp = a.grpsum + (int64_t)b * a.grp_stride;
  unsigned last = 0;
  if (lane == 0) {
    grp[3 * blockIdx.x + 0] = dsz;
    grp[3 * blockIdx.x + 1] = dss;
    grp[3 * blockIdx.x + 2] = dzz;
    __threadfence();
    last = atomicAdd(a.counters + b, 1u) == (unsigned)ngrp - 1u;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  double sums[3];
#pragma unroll 1
  for (int j = 0; j < 3; ++j) warp_tree_arrays_b<1>(grp + j, ngrp, 3, lane, sums + j);
  snapshot(&snap[warp], st, lane);
  if (lane != 0) return;
  a.counters[b] = 0;
  adj_tail(st, snap[warp], sums[0], sums[1], sums[2]);
}

// r' = r + lambda kd for every live problem (gpss.cpp:209) into r[cur^1] and the staging
// matrix the adjoint DMMA reads
__global__ void brupdate_kernel(const BFinArgs a, double* rn) {
  pdl_wait_and_trigger();
  const int b = blockIdx.y;
  const DevState* st = a.st + b;
  if (st->status != RUNNING) return;
  const int cur = st->cur;
  const double lam = st->step;
  const int64_t ob = (int64_t)b * a.ostride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.ostride;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = add(a.vb.r[cur][ob + i], mul(lam, a.vb.kd[ob + i]));
    a.vb.r[cur ^ 1][ob + i] = r;
    rn[ob + i] = r;
  }
}

static int splits_for(int64_t tiles_out, int64_t nblocks, int sm_count) {
  // enough CTAs for ~7 waves of one CTA per SM, splits dividing the reduction evenly
  int s = 1;
  while (s * 2 <= nblocks && tiles_out * s * 2 <= 7LL * sm_count) s *= 2;
  return s;
}

// 16-warp kernels (one CTA per SM): the split count that best fills whole waves, a small
// penalty per split for the partials it adds
static int splits_wide(int64_t tiles_out, int64_t nchunks, int sm_count) {
  int best = 1;
  double best_score = -1.0;
  for (int s = 1; s <= 64 && s <= nchunks; ++s) {
    const int64_t ctas = tiles_out * s;
    const int64_t waves = (ctas + sm_count - 1) / sm_count;
    const double score = (double)ctas / (double)(waves * sm_count) - 0.002 * s;
    if (score > best_score + 1e-12) {
      best_score = score;
      best = s;
    }
  }
  return best;
}

static bool wide_products() {
  static const bool w = [] {
    const char* e = getenv("L1G_DMMA");
    return !(e && std::strcmp(e, "8") == 0);
  }();
  return w;
}
// persistent producer-warp products: one CTA per SM
static int ws_grid(const Op& op) { return op.plan.grid; }
// L1G_BATCH_TAIL=0: no few-live-problems variant beside the compacted products
bool batch_tail_kernels() {
  static const bool on = [] {
    const char* e = getenv("L1G_BATCH_TAIL");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}
// L1G_DMMA=wide: the 16-warp kernels whose consumers issue the copies themselves
static bool ws_products() {
  static const bool w = [] {
    const char* e = getenv("L1G_DMMA");
    return !(e && std::strcmp(e, "wide") == 0);
  }();
  return w;
}

BatchPlan make_batch_plan(const GemvPlan& pl, int B, int sm_count) {
  BatchPlan bp{};
  bp.B = B;
  bp.Bp = (B + BW - 1) / BW * BW;
  const int64_t bz = bp.Bp / BW;
  bp.wide = wide_products();
  if (bp.wide) {  // forward: 32-column chunks; adjoint: row blocks; 128-wide CTA tiles
    bp.fwd_splits = splits_wide((pl.n_pad / 128) * bz, 2 * pl.ncb, sm_count);
    bp.fwd_per = (int)((2 * pl.ncb + bp.fwd_splits - 1) / bp.fwd_splits);
    bp.fwd_splits = (int)((2 * pl.ncb + bp.fwd_per - 1) / bp.fwd_per);
    bp.adj_splits = splits_wide((pl.p_pad / 128) * bz, pl.nrb, sm_count);
    bp.adj_per = (int)((pl.nrb + bp.adj_splits - 1) / bp.adj_splits);
    bp.adj_splits = (int)((pl.nrb + bp.adj_per - 1) / bp.adj_per);
    return bp;
  }
  bp.fwd_splits = splits_for((pl.n_pad / 64) * bz, pl.ncb, sm_count);
  bp.fwd_per = (int)((pl.ncb + bp.fwd_splits - 1) / bp.fwd_splits);
  bp.adj_splits = splits_for(pl.ncb * bz, pl.nrb, sm_count);
  bp.adj_per = (int)((pl.nrb + bp.adj_splits - 1) / bp.adj_splits);
  bp.adj_per = (bp.adj_per + A_RB - 1) / A_RB * A_RB;  // whole stages per split
  return bp;
}

void launch_bfwd(const Op& op, const BatchPlan& bp, const double* D, double* part,
                 cudaStream_t s, const int* active, const int* nact) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(bfwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bfwd_smem()));
  });
  const GemvPlan& pl = op.plan;
  BGemmArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.nrb = pl.nrb;
  a.V = D;
  a.vstride = pl.p_pad;
  a.part = part;
  a.pslab = (int64_t)bp.Bp * pl.n_pad;
  a.ostride = pl.n_pad;
  a.per_split = bp.fwd_per;
  a.nblocks = (int)pl.ncb;
  if (bp.wide) {
    static std::atomic<unsigned long long> wattr{0};
    once_per_device(wattr, [] {
      L1G_CUDA(cudaFuncSetAttribute(bfwd_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bwide_smem()));
      L1G_CUDA(cudaFuncSetAttribute(bfwd_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bwide_smem()));
    });
    const dim3 grid((unsigned)(pl.n_pad / 128), (unsigned)bp.fwd_splits, (unsigned)(bp.Bp / BW));
    if (ws_products()) {
      a.nx = (int)grid.x, a.ny = (int)grid.y, a.nz = (int)grid.z;
      a.active = active, a.nact = nact, a.nb = bp.B;
      a.tail = (nact && batch_tail_kernels()) ? 1 : 0;
      const int items = a.nx * a.ny * a.nz;
      L1G_CUDA(launch_pdl(bfwd_ws_kernel, std::min(items, ws_grid(op)), WP, bwide_smem(), s, a));
      if (a.tail) {
        static std::atomic<unsigned long long> tattr{0};
        once_per_device(tattr, [] {
          L1G_CUDA(cudaFuncSetAttribute(bws_tail_kernel<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)btail_smem()));
        });
        L1G_CUDA(launch_pdl(bws_tail_kernel<false>, std::min(a.nx * a.ny, 2 * ws_grid(op)),
                            T_THREADS, btail_smem(), s, a));
      }
    }
    else L1G_CUDA(launch_pdl(bfwd_wide_kernel, grid, WT, bwide_smem(), s, a));
    return;
  }
  const dim3 grid((unsigned)(pl.n_pad / 64), (unsigned)bp.fwd_splits, (unsigned)(bp.Bp / BW));
  L1G_CUDA(launch_pdl(bfwd_kernel, grid, BT, bfwd_smem(), s, a));
}

void launch_badj(const Op& op, const BatchPlan& bp, const double* R, double* part,
                 cudaStream_t s, const int* active, const int* nact) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(badj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)badj_smem()));
  });
  const GemvPlan& pl = op.plan;
  BGemmArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.nrb = pl.nrb;
  a.V = R;
  a.vstride = pl.n_pad;
  a.part = part;
  a.pslab = (int64_t)bp.Bp * pl.p_pad;
  a.ostride = pl.p_pad;
  a.per_split = bp.adj_per;
  a.nblocks = (int)pl.nrb;
  if (bp.wide) {
    static std::atomic<unsigned long long> wattr{0};
    once_per_device(wattr, [] {
      L1G_CUDA(cudaFuncSetAttribute(badj_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bwide_smem()));
      L1G_CUDA(cudaFuncSetAttribute(badj_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bwide_smem()));
    });
    const dim3 grid((unsigned)(pl.ncb / 2), (unsigned)bp.adj_splits, (unsigned)(bp.Bp / BW));
    if (ws_products()) {
      a.nx = (int)grid.x, a.ny = (int)grid.y, a.nz = (int)grid.z;
      a.active = active, a.nact = nact, a.nb = bp.B;
      a.tail = (nact && batch_tail_kernels()) ? 1 : 0;
      const int items = a.nx * a.ny * a.nz;
      L1G_CUDA(launch_pdl(badj_ws_kernel, std::min(items, ws_grid(op)), WP, bwide_smem(), s, a));
      if (a.tail) {
        static std::atomic<unsigned long long> tattr{0};
        once_per_device(tattr, [] {
          L1G_CUDA(cudaFuncSetAttribute(bws_tail_kernel<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)btail_smem()));
        });
        L1G_CUDA(launch_pdl(bws_tail_kernel<true>, std::min(a.nx * a.ny, 2 * ws_grid(op)),
                            T_THREADS, btail_smem(), s, a));
      }
    }
    else L1G_CUDA(launch_pdl(badj_wide_kernel, grid, WT, bwide_smem(), s, a));
    return;
  }
  const dim3 grid((unsigned)pl.ncb, (unsigned)bp.adj_splits, (unsigned)(bp.Bp / BW));
  L1G_CUDA(launch_pdl(badj_kernel, grid, BT, badj_smem(), s, a));
}

// The live problems of a batch in index order: active[0 .. *nact).  One CTA; the producer-warp
// products read the list right after (same stream, programmatic dependency).
constexpr int BC_T = 256;
__global__ void __launch_bounds__(BC_T) bcompact_kernel(const DevState* st, int B, int* active,
                                                        int* nact) {
  pdl_wait_and_trigger();
  __shared__ int wcnt[BC_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int base = 0;
  for (int b0 = 0; b0 < B; b0 += BC_T) {
    const int b = b0 + threadIdx.x;
    const bool live = b < B && __ldcg(&st[b].status) == RUNNING;
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (lane == 0) wcnt[warp] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < BC_T / 32; ++w) {
      before += w < warp ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    if (live) active[base + before + __popc(m & ((1u << lane) - 1u))] = b;
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nact = base;
}

void launch_bcompact(const DevState* st, int B, int* active, int* nact, cudaStream_t s) {
  L1G_CUDA(launch_pdl(bcompact_kernel, 1, BC_T, 0, s, st, B, active, nact));
}

void launch_bfin(const BFinArgs& a, bool adjoint, int64_t len_pad, cudaStream_t s) {
  const dim3 grid((unsigned)(len_pad / (adjoint ? 64 : 32)), (unsigned)((a.B + BF_W - 1) / BF_W));
  if (adjoint) L1G_CUDA(launch_pdl(bfin_adj_kernel, grid, 32 * BF_W, 0, s, a));
  else L1G_CUDA(launch_pdl(bfin_fwd_kernel, grid, 32 * BF_W, 0, s, a));
}

void launch_brupdate(const BFinArgs& a, double* rn, cudaStream_t s) {
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(a.ostride / 256, 16)),
                  (unsigned)a.B);
  L1G_CUDA(launch_pdl(brupdate_kernel, grid, 256, 0, s, a, rn));
}

}  // namespace l1g
