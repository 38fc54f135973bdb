// gemv.cu -- fused fp64 forward (K d) and adjoint (K^T r) products over the tiled K.
//
// Replaces DenseOperator::do_apply / do_apply_adjoint (linear_operator.hpp:45-48) on the
// GPSS hot path (gpss.cpp:194-196 and :206-211).  Both kernels are persistent (one CTA per
// SM) and warp specialised: warp 0 streams 32x64 K tiles into a 3-stage shared-memory ring
// with cp.async.bulk (TMA engine) + mbarriers; 4*SPLIT consumer warps reduce them, SPLIT
// warps per tile (lane groups own a slice of the tile, a shuffle joins the slices).  Every
// output is the canonical pairwise sum of rounded products (common.cuh), evaluated as
//   per-lane trees inside a tile -> shuffle join -> a binary counter over the tiles of a
//   task -> a tree over task partials, done by the CTA that completes a group last.
// The same completing CTA runs the fused epilogue:
//   forward/ITER : a = (Kx - y)'Kd, b = ||Kd||^2, then the backtracking line search;
//   forward/INIT : r = Kx0 - y, f = ||r||^2;
//   adjoint/ITER : r += lambda Kd (prologue), g' = 2 K^T r, x' = x + lambda d,
//                  s'z, s's, z'z for the next BB step, telemetry, stop tests.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"
#include "steps.cuh"

namespace l1g {

#ifdef L1G_TIMELINE
__device__ unsigned long long g_tl_gemv[256 * 16];
#endif

constexpr int STAGES = 3;
constexpr int TILES_PER_STAGE = 4;
constexpr int DPAD = 16;  // padding of the d slice (doubles), covers d_pos<4>(31)
constexpr int FWD_STAGE_DBL = TILES_PER_STAGE * TILE + 64 + DPAD;
constexpr int ADJ_STAGE_DBL = TILES_PER_STAGE * TILE;
constexpr int FWD_MAX_STAGES = 128;  // column blocks per forward task (counter depth 8)
constexpr int ADJ_MAX_BLOCKS = 16;   // row blocks per adjoint task (counter depth 6)
constexpr int MAX_TR = ADJ_MAX_BLOCKS * TR;
constexpr int RS_PAD = MAX_TR / 8;   // padding of the shared r slice (see rs_pos)

// Finish kernels over a batch of problems (gridDim.y = problems): problem b's partials,
// vectors, state, group sums and counter sit at these offsets from problem 0's.
struct BatchStrides {
  int64_t pstride;  // between consecutive partials of one output
  int64_t bpart, bn, bp, bgrp;
};

struct FwdArgs {
  const double* K;
  int64_t ncb, n_pad;
  int stages, nrg, ncr, mode;
  const double* vin;
  double* vout;
  double* part;
  double* grpsum;
  unsigned* cnt_grp;
  unsigned* cnt_all;
  unsigned* task_ctr;  // sparse forward: dynamic task counter (reset by fwd_finish)
  // sparse forward with the density switch: the support size from which the dense stream
  // runs instead (0: never); it keeps the sparse column ranges, so the finish is the same
  int64_t dense_min;
  DevState* st;
  VecBufs vb;
  BatchStrides bs;     // finish kernels: partial stride, per-problem offsets (blockIdx.y)
  int wpg;             // finish kernels: warps per output group (fin_wpg)
};

struct AdjArgs {
  const double* K;
  int64_t ncb, nrb, p_pad;
  int blocks, ncg, nrr, mode;
  const double* vin;
  double* vout;
  double* part;
  double* grpsum;
  unsigned* cnt_grp;
  unsigned* cnt_all;
  DevState* st;
  VecBufs vb;
  BatchStrides bs;
  int wpg;  // finish kernel: warps per output group (fin_wpg)
  // column shard of a sharded solver (abi.cu): the finish also writes the
  // shard's new x and g and its subtree values of s'z, s's, z'z plus its clock into the
  // allgather packet [x (p_pad) | g (p_pad) | SHARD_SCAL scalars]
  double* pack;
};


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

// Trees over NA interleaved arrays v[i*stride + j], i < count (runtime count, absent beyond),
// by one warp: lane l takes block l of each 32-chunk, the butterfly reduces the chunk, a
// counter joins chunks.  Loads are issued 4 chunks ahead so the L2 latency is paid once
// per 4 chunks instead of once per chunk.
template <int NA>
__device__ __forceinline__ void warp_tree_arrays(const double* v, int count, int stride, int lane,
                                                 double* out) {
  Counter<12> acc[NA];  // chunks < 2^12 per warp block
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
    for (int u = 0; u < 4; ++u) {
      if (c0 + u < chunks) {
#pragma unroll
        for (int j = 0; j < NA; ++j) acc[j].push(warp_tree(x[u][j]), (uint32_t)(c0 + u));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NA; ++j) out[j] = acc[j].final_value((uint32_t)chunks);
}

// position of d unit u (16-byte pair) in the padded per-stage slice: the SPLIT lane groups
// read units u, u + 32/SPLIT, ... at once, which must fall in distinct bank groups
template <int SPLIT>
__device__ __forceinline__ int d_pos(int u) {
  if constexpr (SPLIT == 1) return u;
  else if constexpr (SPLIT == 2) return u + 4 * (u >> 4);
  else return u + 2 * (u >> 3);
}
// position of r[i] in the padded shared r slice (same idea for 8-byte words)
__device__ __forceinline__ int rs_pos(int i) { return i + (i >> 3); }

// ============================================================================ finish kernels
// The finish kernels are chains of dependent memory round trips (partials, vectors, state,
// group sums); every load that does not depend on an earlier one is issued up front.

// canonical tree over partials k in [lo, hi) of one output (p + k * stride), lo a multiple
// of 16 or the block start: chunks of 16 loads in flight at once, each chunk a register tree
// (absent leaves past hi read as +0.0, which leaves every sum unchanged) pushed into the
// binary counter as one level-4 node.  Returns the block value.
template <int L>
__device__ __forceinline__ double tree16(const double (&v)[16]) {
  double t[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) t[i] = add(v[2 * i], v[2 * i + 1]);
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = add(t[2 * i], t[2 * i + 1]);
  return add(add(t[0], t[1]), add(t[2], t[3]));
}
template <int NA>
__device__ __forceinline__ void chunk_trees(const double* p, int64_t stride, int lo, int hi,
                                            double* out) {
  Counter<16> acc[NA];
  for (int k0 = lo; k0 < hi; k0 += 16) {
    const int n = hi - k0 < 16 ? hi - k0 : 16;
    double v[NA][16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (NA == 2) {
        const double2 w = u < n ? __ldcg(reinterpret_cast<const double2*>(p + (int64_t)(k0 + u) * stride))
                                : make_double2(0.0, 0.0);
        v[0][u] = w.x;
        v[NA - 1][u] = w.y;
      } else {
        v[0][u] = u < n ? __ldcg(p + (int64_t)(k0 + u) * stride) : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j].template push_node<4>(tree16<0>(v[j]), (uint32_t)((k0 - lo) >> 4));
  }
  const uint32_t cnt = (uint32_t)(((hi - lo) + 15) & ~15);
#pragma unroll
  for (int j = 0; j < NA; ++j) out[j] = acc[j].final_value(cnt);
}

// the state words, loaded by warp 0 into registers ahead of other loads, stored to shared
constexpr int DS_WORDS = (int)(sizeof(DevState) / 8);
constexpr int DS_PER_LANE = (DS_WORDS + 31) / 32;
__device__ __forceinline__ void state_prefetch(const DevState* st, int lane,
                                               unsigned long long (&w)[DS_PER_LANE]) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(st);
#pragma unroll
  for (int i = 0; i < DS_PER_LANE; ++i) {
    const int j = lane + 32 * i;
    w[i] = j < DS_WORDS ? __ldcg(s + j) : 0ull;
  }
}
__device__ __forceinline__ void state_store(DevState* dst, int lane,
                                            const unsigned long long (&w)[DS_PER_LANE]) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
#pragma unroll
  for (int i = 0; i < DS_PER_LANE; ++i) {
    const int j = lane + 32 * i;
    if (j < DS_WORDS) d[j] = w[i];
  }
  __syncwarp();
}

// One CTA of 8 warps per 32 rows (forward) or 64 columns (adjoint): the task partials of
// each output are split over the warps in aligned power-of-two blocks (a binary counter per
// warp), warp 0 joins the 8 block values pairwise (blocks past the count are absent), runs
// the fused epilogue and reduces its dot-product leaves with the warp butterfly; the CTA
// that counts last joins the group values and runs the scalar part of gp_iterate.
constexpr int FIN_W = 8;
constexpr int FIN_T = 32 * FIN_W;


template <class A>
__device__ __forceinline__ A batch_view(const A& a0, int prob) {
  A a = a0;
  if (prob == 0) return a;
  const BatchStrides& b = a0.bs;
  a.part += prob * b.bpart;
  a.st += prob;
  a.grpsum += prob * b.bgrp;
  a.cnt_all += prob;
  return a;  // vectors: the kernels add prob * bn / bp to a0.vb (runtime-indexed arrays)
}

__device__ __forceinline__ int fin_block(int cnt) {
  int B = 1;
  while (B * FIN_W < cnt) B <<= 1;
  return B;
}

// join of the FIN_W block values of one output held in sv[w][lane] (w < nb present)
__device__ __forceinline__ double fin_join(const double (*sv)[32], int nb, int lane) {
  double x[FIN_W];
#pragma unroll
  for (int w = 0; w < FIN_W; ++w) x[w] = sv[w][lane];
#pragma unroll
  for (int h = 1; h < FIN_W; h <<= 1)
#pragma unroll
    for (int i = 0; i + h < FIN_W; i += 2 * h)
      if (i + h < nb) x[i] = add(x[i], x[i + h]);
  return x[0];
}

// Canonical trees over NA interleaved group arrays (count groups) by a whole CTA of
// FIN_W warps: aligned power-of-two blocks per warp, joined pairwise by warp 0.
template <int NA>
__device__ __forceinline__ void cta_tree_arrays(const double* v, int count, int stride,
                                                double (*sv)[FIN_W][32], double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int B = 32;
  while (B * FIN_W < count) B <<= 1;
  const int lo = warp * B, hi = lo + B < count ? lo + B : count;
  double r[NA];
  if (hi > lo) warp_tree_arrays<NA>(v + (int64_t)lo * stride, hi - lo, stride, lane, r);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NA; ++j) sv[j][warp][0] = hi > lo ? r[j] : 0.0;
  __syncthreads();
  const int nb = (count + B - 1) / B;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    double x[FIN_W];
#pragma unroll
    for (int w = 0; w < FIN_W; ++w) x[w] = sv[j][w][0];
#pragma unroll
    for (int h = 1; h < FIN_W; h <<= 1)
#pragma unroll
      for (int i = 0; i + h < FIN_W; i += 2 * h)
        if (i + h < nb) x[i] = add(x[i], x[i + h]);
    out[j] = x[0];
  }
}

// warps per output group: enough that each warp's aligned block of partials is <= 16 loads
// (all in flight at once); a CTA of FIN_W warps finishes FIN_W / wpg groups
static inline int fin_wpg(int cnt) {
  int w = 1;
  while (w < FIN_W && w * 16 < cnt) w <<= 1;
  return w;
}
__device__ __forceinline__ int fin_block_w(int cnt, int wpg) {
  int B = 1;
  while (B * wpg < cnt) B <<= 1;
  return B;
}
// join of the wpg block values of one output (nb of them present)
__device__ __forceinline__ double fin_join_w(const double (*sv)[32], int wpg, int nb, int lane) {
  double x[FIN_W];
#pragma unroll
  for (int w = 0; w < FIN_W; ++w) x[w] = w < wpg ? sv[w][lane] : 0.0;
#pragma unroll
  for (int h = 1; h < FIN_W; h <<= 1)
#pragma unroll
    for (int i = 0; i + h < FIN_W; i += 2 * h)
      if (i + h < nb) x[i] = add(x[i], x[i + h]);
  return x[0];
}

__global__ void __launch_bounds__(FIN_T) fwd_finish_kernel(const FwdArgs a0) {
  L1G_TL_ENTRY
  pdl_wait_and_trigger();
  L1G_TL_WAITED(a0.mode == FWD_ITER && blockIdx.y == 0, g_tl_gemv, 2, a0.st->k)
  FwdArgs a = batch_view(a0, blockIdx.y);
  if (blockIdx.y && a.vout) a.vout += blockIdx.y * a0.bs.bn;
  const int64_t on = blockIdx.y * a0.bs.bn;
  __shared__ double sv[FIN_W][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpg = a.wpg, gl = warp / wpg, wi = warp - gl * wpg;
  const int ngrp = (int)(a.n_pad / 32);
  const int grp = blockIdx.x * (FIN_W / wpg) + gl;
  const bool live = grp < ngrp;
  const int64_t row = (int64_t)(live ? grp : 0) * 32 + lane;
  // independent loads first: the state words the group leader needs, y or both r buffers
  int status = RUNNING, cur = 0;
  double pre0 = 0.0, pre1 = 0.0;
  if (a.mode != FWD_APPLY) {
    status = __ldcg(&a.st->status);
    if (wi == 0 && live) {
      cur = __ldcg(&a.st->cur);
      if (a.mode == FWD_INIT) {
        pre0 = __ldcg(a0.vb.y + on + row);
      } else {
        pre0 = __ldcg(a0.vb.r[0] + on + row);
        pre1 = __ldcg(a0.vb.r[1] + on + row);
      }
    }
  }
  const int ncr = a.ncr;
  const int B = fin_block_w(ncr, wpg);
  {
    const int lo = wi * B, hi = lo + B < ncr ? lo + B : ncr;
    double bv[1] = {0.0};
    if (live && hi > lo) chunk_trees<1>(a.part + row, a.bs.pstride, lo, hi, bv);
    sv[warp][lane] = bv[0];
    __syncthreads();
  }
  if (status != RUNNING) return;
  if (wi == 0 && live) {
    const double kd = fin_join_w(sv + gl * wpg, wpg, (ncr + B - 1) / B, lane);
    if (a.mode == FWD_APPLY) {
      a.vout[row] = kd;
    } else {
      double l0, l1 = 0.0;
      if (a.mode == FWD_INIT) {
        const double r = sub(kd, pre0);  // Kx0 - y   (gpss.cpp:128)
        a0.vb.r[cur][on + row] = r;
        l0 = mul(r, r);                         // ||r||^2   (gpss.cpp:129)
      } else {
        a0.vb.kd[on + row] = kd;
        l0 = mul(cur ? pre1 : pre0, kd);        // (Kx-y)'Kd (gpss.cpp:195)
        l1 = mul(kd, kd);                       // ||Kd||^2  (gpss.cpp:196)
      }
      l0 = warp_tree(l0);
      l1 = warp_tree(l1);
      if (lane == 0) {
        a.grpsum[2 * grp + 0] = l0;
        a.grpsum[2 * grp + 1] = l1;
        __threadfence();
      }
    }
  }
  if (a.mode == FWD_APPLY) return;
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.cnt_all, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!s_last) return;
  L1G_TL_STAMP(a.mode == FWD_ITER && blockIdx.y == 0 && threadIdx.x == 0, g_tl_gemv, 12, a.st->k)
  __threadfence();
  unsigned long long sw[DS_PER_LANE];
  if (warp == 0) state_prefetch(a.st, lane, sw);  // in flight with the group sums
  __shared__ double tsv[2][FIN_W][32];  // (sv is one array: the tree needs two)
  double AB[2];
  cta_tree_arrays<2>(a.grpsum, ngrp, 2, tsv, AB);
  if (warp != 0) return;
  const double A = AB[0], Bv = AB[1];
  __shared__ DevState s;
  state_store(&s, lane, sw);
  if (lane != 0) return;
  *a.cnt_all = 0;
  if (a.task_ctr) *a.task_ctr = 0;
  fwd_tail(a.st, s, a.mode, A, Bv);
  L1G_TL_STAMP(a.mode == FWD_ITER && blockIdx.y == 0, g_tl_gemv, 13, s.k)
}

__global__ void __launch_bounds__(FIN_T) adj_finish_kernel(const AdjArgs a0) {
  L1G_TL_ENTRY
  pdl_wait_and_trigger();
  L1G_TL_WAITED(a0.mode == ADJ_ITER && blockIdx.y == 0, g_tl_gemv, 4, a0.st->k)
  AdjArgs a = batch_view(a0, blockIdx.y);
  if (blockIdx.y && a.vout) a.vout += blockIdx.y * a0.bs.bp;
  const int64_t ofp = blockIdx.y * a0.bs.bp;
  __shared__ double sv[3][FIN_W][32];  // [2] only for the group-sum tree of the last CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpg = a.wpg, gl = warp / wpg, wi = warp - gl * wpg;
  const int ngrp = (int)(a.p_pad / 64);
  const int grp = blockIdx.x * (FIN_W / wpg) + gl;
  const bool live = grp < ngrp;
  const int64_t col = (int64_t)(live ? grp : 0) * 64 + 2 * lane;
  DevState* st = a.st;
  // independent loads first: state words, and (ITER) x, g of both buffers and d
  int status = RUNNING, cur = 0;
  double lam = 0.0;
  double2 xb[2], gb[2], dd;
  if (a.mode != ADJ_APPLY) {
    status = __ldcg(&st->status);
    if (wi == 0 && live) {
      cur = __ldcg(&st->cur);
      if (a.mode == ADJ_ITER) {
        lam = __ldcg(&st->step);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          xb[b] = __ldcg(reinterpret_cast<const double2*>(a0.vb.x[b] + ofp + col));
          gb[b] = __ldcg(reinterpret_cast<const double2*>(a0.vb.g[b] + ofp + col));
        }
        dd = __ldcg(reinterpret_cast<const double2*>(a0.vb.d + ofp + col));
      } else if (a.pack) {  // ADJ_INIT of a shard: x0 travels with g
        xb[0] = __ldcg(reinterpret_cast<const double2*>(a0.vb.x[cur] + col));
      }
    }
  }
  const int B = fin_block_w(a.nrr, wpg);
  {
    const int lo = wi * B, hi = lo + B < a.nrr ? lo + B : a.nrr;
    double bv[2] = {0.0, 0.0};
    if (live && hi > lo) chunk_trees<2>(a.part + col, a.bs.pstride, lo, hi, bv);
    sv[0][warp][lane] = bv[0];
    sv[1][warp][lane] = bv[1];
    __syncthreads();
  }
  if (status != RUNNING) return;
  if (wi == 0 && live) {
    const int nb = (a.nrr + B - 1) / B;
    const double s0 = fin_join_w(sv[0] + gl * wpg, wpg, nb, lane);
    const double s1 = fin_join_w(sv[1] + gl * wpg, wpg, nb, lane);
    if (a.mode == ADJ_APPLY) {
      *reinterpret_cast<double2*>(a.vout + col) = make_double2(s0, s1);
    } else {
      const double g0 = mul(2.0, s0), g1 = mul(2.0, s1);  // 2 K^T r (gpss.cpp:130, :211)
      if (a.mode == ADJ_INIT) {
        *reinterpret_cast<double2*>(a0.vb.g[cur] + ofp + col) = make_double2(g0, g1);
        if (a.pack) {
          *reinterpret_cast<double2*>(a.pack + col) = xb[0];
          *reinterpret_cast<double2*>(a.pack + a.p_pad + col) = make_double2(g0, g1);
          if (blockIdx.x == 0 && wi == 0 && gl == 0 && lane == 0) {
            double* sc = a.pack + 2 * a.p_pad;
            sc[0] = sc[1] = sc[2] = 0.0;
            sc[3] = elapsed_s(st);
          }
        }
      } else {
        // x' = x + lambda d (gpss.cpp:208), s = x' - x, z = g' - g (gpss.cpp:150-151)
        const double2 xo = cur ? xb[1] : xb[0];
        const double2 go = cur ? gb[1] : gb[0];
        const double x0n = add(xo.x, mul(lam, dd.x)), x1n = add(xo.y, mul(lam, dd.y));
        *reinterpret_cast<double2*>(a0.vb.x[cur ^ 1] + ofp + col) = make_double2(x0n, x1n);
        *reinterpret_cast<double2*>(a0.vb.g[cur ^ 1] + ofp + col) = make_double2(g0, g1);
        if (a.pack) {
          *reinterpret_cast<double2*>(a.pack + col) = make_double2(x0n, x1n);
          *reinterpret_cast<double2*>(a.pack + a.p_pad + col) = make_double2(g0, g1);
        }
        const double sa = sub(x0n, xo.x), sb = sub(x1n, xo.y);
        const double za = sub(g0, go.x), zb = sub(g1, go.y);
        const double dsz = warp_tree(add(mul(sa, za), mul(sb, zb)));
        const double dss = warp_tree(add(mul(sa, sa), mul(sb, sb)));
        const double dzz = warp_tree(add(mul(za, za), mul(zb, zb)));
        if (lane == 0) {
          a.grpsum[3 * grp + 0] = dsz;
          a.grpsum[3 * grp + 1] = dss;
          a.grpsum[3 * grp + 2] = dzz;
          __threadfence();
        }
      }
    }
  }
  if (a.mode != ADJ_ITER) return;
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.cnt_all, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!s_last) return;
  L1G_TL_STAMP(blockIdx.y == 0 && threadIdx.x == 0, g_tl_gemv, 10, st->k)
  __threadfence();
  unsigned long long sw[DS_PER_LANE];
  if (warp == 0) state_prefetch(st, lane, sw);  // in flight with the group sums
  __syncthreads();  // sv is free: the group-sum tree reuses it
  double (*tsv)[FIN_W][32] = reinterpret_cast<double (*)[FIN_W][32]>(&sv[0][0][0]);
  double sums[3];
  cta_tree_arrays<3>(a.grpsum, ngrp, 3, tsv, sums);
  L1G_TL_STAMP(blockIdx.y == 0 && threadIdx.x == 0, g_tl_gemv, 15, st->k)
  if (warp != 0) return;
  const double SZ = sums[0], SS = sums[1], ZZ = sums[2];
  __shared__ DevState s;
  state_store(&s, lane, sw);
  if (lane != 0) return;
  *a.cnt_all = 0;
  if (a.pack) {  // the shard's subtree values; the projection joins them over the ranks
    double* sc = a.pack + 2 * a.p_pad;
    sc[0] = SZ;
    sc[1] = SS;
    sc[2] = ZZ;
    sc[3] = elapsed_s(&s);
  }
  adj_tail(st, s, SZ, SS, ZZ);
  L1G_TL_STAMP(blockIdx.y == 0, g_tl_gemv, 11, s.k)
}

// ============================================================================ forward
// The dense forward stream as a device function: fwd_kernel, and fwd_sparse_kernel when d
// is dense enough (its first 32 * (4 * SPLIT + 1) threads run this, the others return).
template <int SPLIT, int NST = STAGES>
__device__ __forceinline__ void fwd_dense_body(const FwdArgs& a, unsigned char* smem) {
  constexpr int NCONS = 4 * SPLIT;
  constexpr int NQ = 32 / SPLIT;  // column pairs per lane group
  constexpr int RPW = 32 / SPLIT; // rows per warp
  double* sbase = reinterpret_cast<double*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * FWD_STAGE_DBL * 8);
  uint64_t* empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int ntasks = a.nrg * a.ncr;
  if (warp == 0) {  // ---- producer: one elected lane issues every bulk copy
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int rg = t / a.ncr, cr = t - rg * a.ncr;
        const int64_t cb0 = (int64_t)cr * a.stages;
        const int nst = (int)(a.ncb - cb0 < (int64_t)a.stages ? a.ncb - cb0 : (int64_t)a.stages);
        for (int s = 0; s < nst; ++s) {
          mbar_wait(&empty[stage], phase ^ 1u);
          double* dst = sbase + (size_t)stage * FWD_STAGE_DBL;
          mbar_arrive_expect_tx(&full[stage], TILES_PER_STAGE * TILE_BYTES + 512);
#pragma unroll
          for (int w = 0; w < TILES_PER_STAGE; ++w)
            bulk_g2s(dst + w * TILE, a.K + tile_offset(4 * rg + w, cb0 + s, a.ncb), TILE_BYTES,
                     &full[stage]);
          const double* dsrc = a.vin + (cb0 + s) * TC;
          double* ddst = dst + TILES_PER_STAGE * TILE;
#pragma unroll
          for (int g = 0; g < SPLIT; ++g)
            bulk_g2s(ddst + 2 * d_pos<SPLIT>(g * NQ), dsrc + 2 * g * NQ, 512 / SPLIT, &full[stage]);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  // ---- consumers: warp cw -> tile cw / SPLIT (row block 4*rg + tile), row slice
  //      (cw % SPLIT) * RPW + (lane % RPW), column-pair group lane / RPW
  const int cw = warp - 1;
  const int tile = cw / SPLIT;
  const int row = (cw % SPLIT) * RPW + (lane % RPW);  // row inside the tile
  const int qg = lane / RPW;                           // column-pair group
  int stage = 0;
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const int rg = t / a.ncr, cr = t - rg * a.ncr;
    const int64_t cb0 = (int64_t)cr * a.stages;
    const int nst = (int)(a.ncb - cb0 < (int64_t)a.stages ? a.ncb - cb0 : (int64_t)a.stages);
    Counter<8> acc;
    for (int s = 0; s < nst; ++s) {
      mbar_wait(&full[stage], phase);
      const double* sb = sbase + (size_t)stage * FWD_STAGE_DBL;
      const double* kt = sb + tile * TILE;
      const double2* du = reinterpret_cast<const double2*>(sb + TILES_PER_STAGE * TILE);
      double v = tree<NQ>([&](int k) {
        const int q = qg * NQ + k;
        const int o = 64 * q + (row ^ (q & 15));  // in_tile(row, 2q); column 2q+1 is 32 later
        const double2 d = du[d_pos<SPLIT>(q)];
        return add(mul(kt[o], d.x), mul(kt[o + 32], d.y));
      });
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      // join the SPLIT column slices of the row: adjacent groups are adjacent subtrees
#pragma unroll
      for (int o = RPW; o < 32; o <<= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
      acc.push(v, (uint32_t)s);
      if (++stage == NST) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (qg == 0) {
      const int64_t grow = (int64_t)rg * ROW_GROUP + tile * TR + row;
      a.part[(int64_t)cr * a.n_pad + grow] = acc.final_value((uint32_t)nst);
    }
  }
}

template <int SPLIT>
__global__ void __launch_bounds__(32 * (4 * SPLIT + 1), 1) fwd_kernel(const FwdArgs a) {
  pdl_wait_and_trigger();
  if (a.mode != FWD_APPLY && a.st->status != RUNNING) return;
  extern __shared__ __align__(128) unsigned char smem[];
  fwd_dense_body<SPLIT>(a, smem);
}


// ============================================================================ adjoint
template <int SPLIT>
__global__ void __launch_bounds__(32 * (4 * SPLIT + 1), 1) adj_kernel(const AdjArgs a) {
  constexpr int NCONS = 4 * SPLIT;
  constexpr int NQ = 32 / SPLIT;  // column pairs per warp
  constexpr int RPL = 32 / SPLIT; // rows per lane group
  extern __shared__ __align__(128) unsigned char smem[];
  double* sbase = reinterpret_cast<double*>(smem);
  double* vslot = sbase + (size_t)STAGES * ADJ_STAGE_DBL;         // [2][2][MAX_TR] r, kd
  double* rs = vslot + 4 * MAX_TR;                                 // padded r_new slice
  uint64_t* full = reinterpret_cast<uint64_t*>(rs + MAX_TR + RS_PAD);
  uint64_t* empty = full + STAGES;
  uint64_t* vfull = empty + STAGES;  // [2]
  uint64_t* vempty = vfull + 2;      // [2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int ntasks = a.ncg * a.nrr;
  // K is immutable: the first ring stages of this CTA's first task are requested before
  // waiting for the preceding grid (PDL), so the ring fill overlaps the previous kernel.
  L1G_TL_ENTRY
  int npre = 0;
  if (threadIdx.x == 0 && (int)blockIdx.x < ntasks) {
    const int t = blockIdx.x;
    const int cg = t / a.nrr, rr = t - cg * a.nrr;
    const int64_t rb0 = (int64_t)rr * a.blocks;
    const int nb = (int)(a.nrb - rb0 < (int64_t)a.blocks ? a.nrb - rb0 : (int64_t)a.blocks);
    npre = nb < STAGES ? nb : STAGES;
    for (int s = 0; s < npre; ++s) {
      mbar_arrive_expect_tx(&full[s], TILES_PER_STAGE * TILE_BYTES);
      bulk_g2s(sbase + (size_t)s * ADJ_STAGE_DBL, a.K + tile_offset(rb0 + s, 4 * (int64_t)cg, a.ncb),
               TILES_PER_STAGE * TILE_BYTES, &full[s]);
    }
  }
  pdl_wait_and_trigger();
  L1G_TL_WAITED(a.mode == ADJ_ITER, g_tl_gemv, 3, a.st->k)
  if (a.mode != ADJ_APPLY && a.st->status != RUNNING) {
    for (int s = 0; s < npre; ++s) mbar_wait(&full[s], 0);  // no copy outlives the CTA
    return;
  }
  const int64_t tr = (int64_t)a.blocks * TR;
  const int cur = (a.mode == ADJ_APPLY) ? 0 : a.st->cur;
  const double* rin = (a.mode == ADJ_APPLY) ? a.vin : a.vb.r[cur];
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int j = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++j) {
        const int cg = t / a.nrr, rr = t - cg * a.nrr;
        const int64_t rb0 = (int64_t)rr * a.blocks;
        const int nb = (int)(a.nrb - rb0 < (int64_t)a.blocks ? a.nrb - rb0 : (int64_t)a.blocks);
        const int64_t row0 = rr * tr;
        // the task's slices of r (and Kd) into vector slot j&1
        if (j >= 2) mbar_wait(&vempty[j & 1], (uint32_t)(((j - 2) >> 1) & 1));
        double* vs = vslot + (j & 1) * 2 * MAX_TR;
        const uint32_t vbytes = (uint32_t)(nb * TR * 8);
        mbar_arrive_expect_tx(&vfull[j & 1], a.mode == ADJ_ITER ? 2 * vbytes : vbytes);
        bulk_g2s(vs, rin + row0, vbytes, &vfull[j & 1]);
        if (a.mode == ADJ_ITER) bulk_g2s(vs + MAX_TR, a.vb.kd + row0, vbytes, &vfull[j & 1]);
        for (int s = 0; s < nb; ++s) {
          if (j > 0 || s >= npre) {  // (the first npre stages were issued before the wait)
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&full[stage], TILES_PER_STAGE * TILE_BYTES);
            bulk_g2s(sbase + (size_t)stage * ADJ_STAGE_DBL,
                     a.K + tile_offset(rb0 + s, 4 * (int64_t)cg, a.ncb),
                     TILES_PER_STAGE * TILE_BYTES, &full[stage]);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  // consumers: warp cw -> tile cw / SPLIT (column block 4*cg + tile), column pair
  // (cw % SPLIT) * NQ + (lane % NQ), row slice lane / NQ
  const int cw = warp - 1, ct = threadIdx.x - 32;
  const int tile = cw / SPLIT;
  const int q = (cw % SPLIT) * NQ + (lane % NQ);
  const int rgp = lane / NQ;
  const double lam = (a.mode == ADJ_ITER) ? a.st->step : 0.0;
  int stage = 0;
  uint32_t phase = 0;
  int j = 0;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x, ++j) {
    const int cg = t / a.nrr, rr = t - cg * a.nrr;
    const int64_t rb0 = (int64_t)rr * a.blocks;
    const int nb = (int)(a.nrb - rb0 < (int64_t)a.blocks ? a.nrb - rb0 : (int64_t)a.blocks);
    const int64_t row0 = rr * tr;
    // the task's slice of r (ITER: r + lambda Kd, gpss.cpp:209) from the staged slot
    mbar_wait(&vfull[j & 1], (uint32_t)((j >> 1) & 1));
    const double* vs = vslot + (j & 1) * 2 * MAX_TR;
    named_bar_sync(1, 32 * NCONS);  // previous task's readers of rs are done
    for (int i = ct; i < nb * TR; i += 32 * NCONS) {
      double r = vs[i];
      if (a.mode == ADJ_ITER) {
        r = add(r, mul(lam, vs[MAX_TR + i]));
        if (cg == 0) a.vb.r[cur ^ 1][row0 + i] = r;
      }
      rs[rs_pos(i)] = r;
    }
    named_bar_sync(1, 32 * NCONS);
    __syncwarp();
    if (lane == 0) mbar_arrive(&vempty[j & 1]);
    Counter<6> acc0, acc1;
    for (int s = 0; s < nb; ++s) {
      mbar_wait(&full[stage], phase);
      const double* kt = sbase + (size_t)stage * ADJ_STAGE_DBL + tile * TILE;
      const int rbase = s * TR + rgp * RPL;
      double2 v = tree2<RPL>([&](int k) {
        const int i = rgp * RPL + k;
        const int o = 64 * q + (i ^ (q & 15));  // in_tile(i, 2q); column 2q+1 is 32 later
        const double r = rs[rs_pos(rbase + k)];
        return make_double2(mul(kt[o], r), mul(kt[o + 32], r));
      });
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
#pragma unroll
      for (int o = NQ; o < 32; o <<= 1) {
        v.x = add(v.x, __shfl_xor_sync(0xffffffffu, v.x, o));
        v.y = add(v.y, __shfl_xor_sync(0xffffffffu, v.y, o));
      }
      acc0.push(v.x, (uint32_t)s);
      acc1.push(v.y, (uint32_t)s);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (rgp == 0) {
      const int64_t col = (int64_t)cg * COL_GROUP + tile * TC + 2 * q;
      *reinterpret_cast<double2*>(a.part + (int64_t)rr * a.p_pad + col) =
          make_double2(acc0.final_value((uint32_t)nb), acc1.final_value((uint32_t)nb));
    }
  }
}

// ============================================================================ sparse forward
// K d for a direction with few nonzeros (gpss.cpp:194: d = h - x, and both h and x live on
// the l1 ball, so d is supported on a small fraction of the columns).  The canonical value
// is unchanged: a column with d_j = 0 contributes an exact-zero leaf and fl(s + 0) = s, so
// the pairwise tree over all columns equals the tree over the support with the same nesting
// (bit for bit, up to the sign of an exactly-zero result; K is finite).
//
// Task = (32 row blocks = 1024 rows, aligned column range of <= 1024 columns), handed out
// dynamically.  Warp 0 turns the range's support bitmap (written by proj_kernel) into a
// schedule in shared memory (double-buffered across tasks): per support column its offset
// in the tiled K, d_j, and its fold step.  The fold is the same for every row: leaf k meets
// its right neighbour at level l_k = bitlength(j_k ^ j_{k+1}) (j = column offset in the
// range), so it first absorbs the pending groups below l_k (increasing level order), then
// waits in slot l_k; the last leaf absorbs everything.  The open-slot sets come from a warp
// scan over the maps v -> (v & ~low(l_k)) | bit(l_k), which compose associatively.
// Consumer warp w owns row blocks 2w, 2w+1 of the task (lane = a row in each; the fold
// control is shared) and streams their 256-byte column runs straight from HBM with a
// SP_PF-deep register prefetch; slots live in shared memory.
// Range partials go to the dense kernel's buffer, so fwd_finish_kernel is shared.
#ifndef L1G_SP_NCW
#define L1G_SP_NCW 16
#endif
#ifndef L1G_SP_PF
#define L1G_SP_PF 16
#endif
#ifndef L1G_FWD_DENSE_FRAC_DEFAULT
#define L1G_FWD_DENSE_FRAC_DEFAULT 0.8
#endif
constexpr int SP_NCW = L1G_SP_NCW;  // consumer warps
constexpr int SP_RPW = 2;      // row blocks per consumer warp (lane = one row in each)
constexpr int SP_RB = SP_NCW * SP_RPW;  // row blocks per task
constexpr int SP_NT = SP_NCW * 32 * SP_RPW;  // slot columns (one per row)
constexpr int SP_MAXT = 16;    // tiles per range (<= 1024 columns, levels 1..10)
constexpr int SP_W = SP_MAXT * TC;
constexpr int SP_LVLS = 11;
constexpr int SP_PF = L1G_SP_PF;  // loads in flight per consumer thread and row
struct SpEnt {
  int coff;  // (tile column block) * TILE + j * 32
  int meta;  // [0,5) level (31 = last leaf), [5,9) column swizzle, [9,20) open slots absorbed
  double d;
};
struct SpInfo {
  int task, count;
};
static size_t sp_smem_own() {
  return (size_t)2 * SP_W * sizeof(SpEnt) + (size_t)SP_LVLS * SP_NT * 8 + 2 * sizeof(SpInfo) +
         4 * 8 + 16;
}
// the sparse kernel also hosts the dense stream (density switch), with a 2-stage ring so
// the kernel's shared memory stays near its own 122 KB
constexpr int SP_DENSE_STAGES = 2;
static size_t sp_smem() {
  return std::max(sp_smem_own(),
                  (size_t)SP_DENSE_STAGES * FWD_STAGE_DBL * 8 + 2 * SP_DENSE_STAGES * 8);
}

__global__ void __launch_bounds__(32 * (SP_NCW + 1), 1) fwd_sparse_kernel(const FwdArgs a) {
  L1G_TL_ENTRY
  pdl_wait_and_trigger();
  L1G_TL_WAITED(true, g_tl_gemv, 1, a.st->k)
  const int status = __ldcg(&a.st->status);
  const int64_t dsup = a.dense_min > 0 ? __ldcg(&a.st->dsup) : 0;  // both loads in flight
  if (status != RUNNING) return;
  extern __shared__ __align__(128) unsigned char smem[];
  if (a.dense_min > 0 && dsup >= a.dense_min) {
    // dense d: the TMA stream over all of K beats the gather; same column ranges (and tree)
    if (threadIdx.x >= 32 * 5) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&a.st->prof[23], 1.0);  // telemetry
    fwd_dense_body<1, SP_DENSE_STAGES>(a, smem);
    return;
  }
  SpEnt* ent = reinterpret_cast<SpEnt*>(smem);  // [2][SP_W]
  double* slots = reinterpret_cast<double*>(ent + 2 * SP_W);
  SpInfo* info = reinterpret_cast<SpInfo*>(slots + (size_t)SP_LVLS * SP_NT);
  uint64_t* sfull = reinterpret_cast<uint64_t*>(info + 2) + 1;  // 8-byte aligned
  uint64_t* sempty = sfull + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], SP_NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t nrb = a.n_pad / TR;
  const int64_t nrq = (nrb + SP_RB - 1) / SP_RB;
  const int ntasks = (int)(nrq * a.ncr);
  if (warp == 0) {  // ---- schedule builder
    const uint64_t* mask = reinterpret_cast<const uint64_t*>(a.vb.dmask);
    for (int it = 0;; ++it) {
      const int bb = it & 1;
      mbar_wait(&sempty[bb], (uint32_t)(((it >> 1) & 1) ^ 1));
      int t = 0;
      if (lane == 0) t = (int)atomicAdd(a.task_ctr, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntasks) {
        if (lane == 0) {
          info[bb].task = -1;
          mbar_arrive(&sfull[bb]);
        }
        break;
      }
      const int rq = t / a.ncr, cr = t - rq * a.ncr;
      const int64_t cb0 = (int64_t)cr * a.stages;
      const int nst = (int)(a.ncb - cb0 < (int64_t)a.stages ? a.ncb - cb0 : (int64_t)a.stages);
      uint64_t w = lane < nst ? __ldg(mask + cb0 + lane) : 0ull;
      const int cnt = __popcll(w);
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int total = __shfl_sync(0xffffffffu, inc, 31);
      SpEnt* e = ent + bb * SP_W;
      {  // column offsets, in column order
        int pos = inc - cnt;
        const int cbase = (int)((cb0 + lane) * TILE);
        while (w) {
          const int j = __ffsll((long long)w) - 1;
          w &= w - 1;
          e[pos++].coff = cbase + j * TR;
        }
      }
      __syncwarp();
      // fold steps, 32 leaves at a time; open-slot set carried across chunks
      unsigned carry = 0;
      for (int k0 = 0; k0 < total; k0 += 32) {
        const int k = k0 + lane;
        int lvl = 31, sw = 0, jr = 0;
        double dv = 0.0;
        if (k < total) {
          const int co = e[k].coff;
          const int cbk = co / TILE, j = (co - cbk * TILE) / TR;
          jr = (int)(cbk - cb0) * TC + j;
          sw = col_swz(j);
          dv = __ldg(a.vin + (int64_t)cbk * TC + j);
          if (k + 1 < total) {
            const int cn = e[k + 1].coff;
            const int cbn = cn / TILE, jn = (cn - cbn * TILE) / TR;
            lvl = 32 - __clz(jr ^ ((int)(cbn - cb0) * TC + jn));
          }
        }
        const unsigned low = (1u << lvl) - 1u;
        // map f(v) = (v & M) | B; inclusive scan of compositions (earlier maps first)
        unsigned M = k < total ? ~low : ~0u, B = (k < total && lvl < 31) ? (1u << lvl) : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned Mp = __shfl_up_sync(0xffffffffu, M, o);
          const unsigned Bp = __shfl_up_sync(0xffffffffu, B, o);
          if (lane >= o) {  // f_this o f_prev
            B = (Bp & M) | B;
            M = Mp & M;
          }
        }
        // open set before leaf k: apply the exclusive prefix to carry
        unsigned Mx = __shfl_up_sync(0xffffffffu, M, 1), Bx = __shfl_up_sync(0xffffffffu, B, 1);
        if (lane == 0) {
          Mx = ~0u;
          Bx = 0u;
        }
        const unsigned open = (carry & Mx) | Bx;
        if (k < total) {
          e[k].meta = lvl | (sw << 5) | (int)((open & low) << 9);
          e[k].d = dv;
        }
        carry = (carry & __shfl_sync(0xffffffffu, M, 31)) | __shfl_sync(0xffffffffu, B, 31);
      }
      if (rq == 0) {  // telemetry: support columns streamed (proj_profile [18], [19])
        if (lane == 0) {
          atomicAdd(&a.st->prof[18], (double)total);
          if (cr == 0) atomicAdd(&a.st->prof[19], 1.0);
        }
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) {
        info[bb].task = t;
        info[bb].count = total;
        mbar_arrive(&sfull[bb]);
      }
    }
    return;
  }
  // ---- consumers
  const int cw = warp - 1;
  double* my0 = slots + cw * 64 + lane;  // slot l of row (block 2cw, lane) at my0[l * SP_NT]
  double* my1 = my0 + 32;                // row (block 2cw + 1, lane)
  const int64_t rbs = a.ncb * TILE;      // one row block further in K
  for (int it = 0;; ++it) {
    const int bb = it & 1;
    mbar_wait(&sfull[bb], (uint32_t)((it >> 1) & 1));
    const int t = info[bb].task;
    if (t < 0) break;
    const int L = info[bb].count;
    const int rq = t / a.ncr, cr = t - rq * a.ncr;
    const int64_t rb = (int64_t)rq * SP_RB + SP_RPW * cw;
    const bool live0 = rb < nrb, live1 = rb + 1 < nrb;
    const double* kr0 = a.K + tile_offset(live0 ? rb : nrb - 1, 0, a.ncb);
    const double* kr1 = live1 ? kr0 + rbs : kr0;
    const SpEnt* e = ent + bb * SP_W;
    double kv0[SP_PF], kv1[SP_PF];
#pragma unroll
    for (int u = 0; u < SP_PF; ++u) {
      if (u < L) {
        const int o = e[u].coff + (lane ^ ((e[u].meta >> 5) & 15));
        kv0[u] = __ldcs(kr0 + o);
        kv1[u] = __ldcs(kr1 + o);
      }
    }
    double x0 = 0.0, x1 = 0.0;
    for (int k0 = 0; k0 < L; k0 += SP_PF) {
#pragma unroll
      for (int u = 0; u < SP_PF; ++u) {
        const int k = k0 + u;
        if (k >= L) break;
        const int meta = e[k].meta;
        const double dk = e[k].d;
        x0 = mul(kv0[u], dk);
        x1 = mul(kv1[u], dk);
        const int kn = k + SP_PF;
        if (kn < L) {
          const int o = e[kn].coff + (lane ^ ((e[kn].meta >> 5) & 15));
          kv0[u] = __ldcs(kr0 + o);
          kv1[u] = __ldcs(kr1 + o);
        }
        unsigned pm = (unsigned)meta >> 9;
        while (pm) {
          const int lv = (__ffs(pm) - 1) * SP_NT;
          x0 = add(my0[lv], x0);
          x1 = add(my1[lv], x1);
          pm &= pm - 1;
        }
        const int lvl = meta & 31;
        if (lvl < 31) {
          my0[lvl * SP_NT] = x0;
          my1[lvl * SP_NT] = x1;
        }
      }
    }
    double* po = a.part + (int64_t)cr * a.n_pad + rb * TR + lane;
    if (live0) po[0] = x0;
    if (live1) po[TR] = x1;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sempty[bb]);
  }
}

// ============================================================================ host side
static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

GemvPlan make_plan(int64_t n, int64_t p, int sm_count) {
  GemvPlan pl{};
  pl.n = n;
  pl.p = p;
  pl.n_pad = cdiv(n > 0 ? n : 1, ROW_GROUP) * ROW_GROUP;
  pl.p_pad = cdiv(p > 0 ? p : 1, COL_GROUP) * COL_GROUP;
  pl.nrb = pl.n_pad / TR;
  pl.ncb = pl.p_pad / TC;
  pl.nrg = (int)(pl.n_pad / ROW_GROUP);
  pl.ncg = (int)(pl.p_pad / COL_GROUP);
  const int64_t target = 8LL * sm_count;
  int s = FWD_MAX_STAGES;
  while (s > 1 && (s > pl.ncb || pl.nrg * cdiv(pl.ncb, s) < target)) s >>= 1;
  pl.fwd_stages = s;
  pl.ncr = (int)cdiv(pl.ncb, s);
  int b = ADJ_MAX_BLOCKS;
  while (b > 1 && (b > pl.nrb || pl.ncg * cdiv(pl.nrb, b) < target)) b >>= 1;
  pl.adj_blocks = b;
  pl.nrr = (int)cdiv(pl.nrb, b);
  // sparse forward: ranges of <= 1024 columns, narrower when that leaves SMs idle
  const int64_t nrq = cdiv(pl.nrb, SP_RB);
  static const int sp_waves = [] {
    const char* e = getenv("L1G_SP_WAVES");
    const int v = e ? atoi(e) : 3;
    return v > 0 ? v : 3;
  }();
  int t = SP_MAXT;
  while (t > 1 && nrq * cdiv(pl.ncb, t) < (int64_t)sp_waves * sm_count) t >>= 1;
  pl.sp_tiles = t;
  pl.sp_ncr = (int)cdiv(pl.ncb, t);
  // density switch: from this fraction of nonzero columns in d the dense stream (6.5 TB/s over
  // all of K) beats the gather over the support columns (L1G_FWD_DENSE_FRAC; <= 0 disables)
  static const double dense_frac = [] {
    const char* e = getenv("L1G_FWD_DENSE_FRAC");
    return e ? atof(e) : L1G_FWD_DENSE_FRAC_DEFAULT;
  }();
  pl.dense_min = dense_frac > 0.0 ? std::max<int64_t>(1, (int64_t)std::ceil(dense_frac * (double)p)) : 0;
  pl.grid = sm_count;
  return pl;
}

static size_t fwd_smem() { return (size_t)STAGES * FWD_STAGE_DBL * 8 + 2 * STAGES * 8; }
static size_t adj_smem() {
  return (size_t)STAGES * ADJ_STAGE_DBL * 8 + (4 * MAX_TR + MAX_TR + RS_PAD) * 8 +
         (2 * STAGES + 4) * 8;
}

static int split_choice() {
  static int s = [] {
    const char* e = getenv("L1G_SPLIT");
    const int v = e ? atoi(e) : 1;
    return (v == 1 || v == 2 || v == 4) ? v : 1;
  }();
  return s;
}

template <int SPLIT>
static void fwd_main_launch(const FwdArgs& a, int grid, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(fwd_kernel<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)fwd_smem()));
  });
  L1G_CUDA(launch_pdl(fwd_kernel<SPLIT>, grid, 32 * (4 * SPLIT + 1), fwd_smem(), s, a));
}

template <int SPLIT>
static void adj_main_launch(const AdjArgs& a, int grid, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(adj_kernel<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)adj_smem()));
  });
  L1G_CUDA(launch_pdl(adj_kernel<SPLIT>, grid, 32 * (4 * SPLIT + 1), adj_smem(), s, a));
}

static FwdArgs fwd_args(const Op& op, const Workspace& ws, int mode, const double* vin,
                        double* vout, const VecBufs* vb, DevState* st) {
  const GemvPlan& pl = op.plan;
  FwdArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.n_pad = pl.n_pad;
  a.stages = pl.fwd_stages;
  a.nrg = pl.nrg;
  a.ncr = pl.ncr;
  a.mode = mode;
  a.vin = vin;
  a.vout = vout;
  a.part = ws.fwd_part;
  a.grpsum = ws.grpsum;
  a.cnt_grp = ws.counters;
  a.cnt_all = ws.counters + pl.nrg + pl.ncg;
  a.st = st;
  if (vb) a.vb = *vb;
  a.bs.pstride = pl.n_pad;
  return a;
}

static AdjArgs adj_args(const Op& op, const Workspace& ws, int mode, const double* vin,
                        double* vout, const VecBufs* vb, DevState* st) {
  const GemvPlan& pl = op.plan;
  AdjArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.nrb = pl.nrb;
  a.p_pad = pl.p_pad;
  a.blocks = pl.adj_blocks;
  a.ncg = pl.ncg;
  a.nrr = pl.nrr;
  a.mode = mode;
  a.vin = vin;
  a.vout = vout;
  a.part = ws.adj_part;
  a.grpsum = ws.grpsum;
  a.cnt_grp = ws.counters + pl.nrg;
  a.cnt_all = ws.counters + pl.nrg + pl.ncg + 1;
  a.st = st;
  if (vb) a.vb = *vb;
  a.bs.pstride = pl.p_pad;
  return a;
}

// main forward kernel over the operator's columns -> range partials in ws.fwd_part;
// returns the args the finish kernel needs (range count / widths)
static FwdArgs fwd_main(const Op& op, const Workspace& ws, FwdArgs a, const uint32_t* dmask,
                        bool sparse, cudaStream_t s, bool dense_switch = false) {
  const GemvPlan& pl = op.plan;
  if (sparse && dmask) {
    a.dense_min = (dense_switch && a.mode == FWD_ITER) ? pl.dense_min : 0;
    static std::atomic<unsigned long long> attr{0};
    once_per_device(attr, [] {
      L1G_CUDA(cudaFuncSetAttribute(fwd_sparse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sp_smem()));
    });
    a.vb.dmask = const_cast<uint32_t*>(dmask);
    a.stages = pl.sp_tiles;
    a.ncr = pl.sp_ncr;
    a.task_ctr = ws.counters + pl.nrg + pl.ncg + 2;
    const int64_t ntasks = (pl.nrb + SP_RB - 1) / SP_RB * pl.sp_ncr;
    L1G_CUDA(launch_pdl(fwd_sparse_kernel, (int)std::min<int64_t>(pl.grid, ntasks),
                        32 * (SP_NCW + 1), sp_smem(), s, a));
    return a;
  }
  const int grid = (int)std::min<int64_t>(pl.grid, (int64_t)pl.nrg * pl.ncr);
  switch (split_choice()) {
    case 1: fwd_main_launch<1>(a, grid, s); break;
    case 4: fwd_main_launch<4>(a, grid, s); break;
    default: fwd_main_launch<2>(a, grid, s); break;
  }
  return a;
}

static void adj_main(const Op& op, const AdjArgs& a, cudaStream_t s) {
  const GemvPlan& pl = op.plan;
  const int grid = (int)std::min<int64_t>(pl.grid, (int64_t)pl.ncg * pl.nrr);
  switch (split_choice()) {
    case 1: adj_main_launch<1>(a, grid, s); break;
    case 4: adj_main_launch<4>(a, grid, s); break;
    default: adj_main_launch<2>(a, grid, s); break;
  }
}

static void fin_launch(FwdArgs a, cudaStream_t s) {
  a.wpg = fin_wpg(a.ncr);
  const int64_t ngrp = a.n_pad / 32, gpc = FIN_W / a.wpg;
  L1G_CUDA(launch_pdl(fwd_finish_kernel, (int)((ngrp + gpc - 1) / gpc), FIN_T, 0, s, a));
}
static void fin_launch(AdjArgs a, cudaStream_t s) {
  a.wpg = fin_wpg(a.nrr);
  const int64_t ngrp = a.p_pad / 64, gpc = FIN_W / a.wpg;
  L1G_CUDA(launch_pdl(adj_finish_kernel, (int)((ngrp + gpc - 1) / gpc), FIN_T, 0, s, a));
}

void launch_fwd(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout,
                const VecBufs* vb, DevState* st, cudaStream_t s, bool sparse, bool dense_switch) {
  FwdArgs a = fwd_args(op, ws, mode, (mode == FWD_ITER) ? vb->d : vin, vout, vb, st);
  a = fwd_main(op, ws, a, a.vb.dmask, sparse && mode == FWD_ITER, s, dense_switch);
  fin_launch(a, s);
}

// gp_init from x0 = 0 (gpss.cpp:126-129): K x0 is exactly zero (each product is +-0 and so
// is every pairwise sum; r = +-0 - y = -y either way), so the forward pass over K is skipped
// and the finish runs on one zero partial per row -- the same r, f and state as the full
// product.  The matvec is still counted by the caller (test_gpss.cpp:366-375).
void launch_fwd_init_zero(const Op& op, const Workspace& ws, const VecBufs* vb, DevState* st,
                          cudaStream_t s) {
  FwdArgs a = fwd_args(op, ws, FWD_INIT, nullptr, nullptr, vb, st);
  a.ncr = 1;
  L1G_CUDA(cudaMemsetAsync(ws.fwd_part, 0, (size_t)op.plan.n_pad * sizeof(double), s));
  fin_launch(a, s);
}

void launch_adj(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout,
                const VecBufs* vb, DevState* st, cudaStream_t s, double* pack) {
  AdjArgs a = adj_args(op, ws, mode, vin, vout, vb, st);
  a.pack = pack;
  adj_main(op, a, s);
  fin_launch(a, s);
}

// ---- column-sharded pieces: rank partials and their combination
void launch_fwd_part(const Op& op, const Workspace& ws, const double* vin, const uint32_t* dmask,
                     bool sparse, double* out, DevState* st, cudaStream_t s) {
  FwdArgs a = fwd_args(op, ws, FWD_APPLY, vin, out, nullptr, st);
  a = fwd_main(op, ws, a, dmask, sparse, s);
  a.mode = FWD_APPLY;  // the finish only writes the shard's tree values
  fin_launch(a, s);
}

void launch_fwd_combine(const Op& op, const Workspace& ws, int mode, const double* recv, int nr,
                        const VecBufs* vb, DevState* st, cudaStream_t s) {
  FwdArgs a = fwd_args(op, ws, mode, nullptr, nullptr, vb, st);
  a.part = const_cast<double*>(recv);
  a.ncr = nr;
  a.task_ctr = ws.counters + op.plan.nrg + op.plan.ncg + 2;
  fin_launch(a, s);
}

}  // namespace l1g

#ifdef L1G_TIMELINE
extern "C" int l1g_debug_timeline_gemv(unsigned long long* out4096, int reset) {
  if (reset) {
    static unsigned long long ones[256 * 16];
    for (auto& v : ones) v = ~0ull;
    return (int)cudaMemcpyToSymbol(l1g::g_tl_gemv, ones, sizeof(ones));
  }
  return (int)cudaMemcpyFromSymbol(out4096, l1g::g_tl_gemv, sizeof(unsigned long long) * 256 * 16);
}
#endif
