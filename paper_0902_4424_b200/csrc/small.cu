// small.cu -- one gp_iterate step after the projection (gpss.cpp:194-217) for problems whose
// K fits in one thread-block cluster's shared memory (n_pad <= 384, p_pad <= 1024: BASELINE
// C1 and smaller), as ONE kernel instead of the four of the large path (forward product,
// forward finish with the backtracking line search, adjoint, adjoint finish with the step and
// the secant dots).  On an L2-resident 2 MB operator those four cost ~22 us per iteration in
// kernel boundaries and dependent round trips; here the cluster keeps its K tiles in shared
// memory and joins its partial sums through distributed shared memory.
//
// CTA r of the cluster owns column tile r (64 columns) of K: every tree below is the
// canonical pairwise tree of the large path (common.cuh), so the results are the same bits:
//   K d   per row: the 64-column tile subtree (tree over 32 column pairs, fwd_kernel) in each
//         CTA, then the tiles pairwise in column order (absent tiles past the end);
//   a, b  per 32-row group a warp tree, then the groups pairwise (fwd_finish);
//   K^T r' per column: 32-row tile subtrees, then the tiles pairwise (adj_kernel / finish);
//   s'z, s's, z'z  per 64-column group a warp tree over column pairs, then the groups
//         pairwise (adj_finish).
// Every CTA computes K d, a, b and the line search itself (same inputs, same bits), so
// nothing but the tile partials and the three group sums crosses the cluster.
#include <cooperative_groups.h>

#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"
#include "steps.cuh"

namespace cg = cooperative_groups;

namespace l1g {

constexpr int SMALL_T = 512;
constexpr int SMALL_MAX_RB = 12;  // n_pad <= 384
constexpr int SMALL_MAX_CS = 16;  // p_pad <= 1024

struct SmallArgs {
  const double* K;
  int64_t ncb;
  int nrb, cs;
  DevState* st;
  VecBufs vb;
};

struct SmallShared {
  double kdp[SMALL_MAX_RB * TR];    // this CTA's tile value of K d, per row
  double kd[SMALL_MAX_RB * TR];     // K d (joined over the cluster)
  double rn[SMALL_MAX_RB * TR];     // r' = r + lambda K d
  double colp[16][TC];              // adjoint: per row tile, per column of this CTA
  double grp[2][16];                // a, b per 32-row group
  double gsum[SMALL_MAX_CS][3];     // CTA 0: the CTAs' s'z, s's, z'z group values
  double dv[TC];
  double lam;
  int ok;
  uint64_t kbar;
  DevState s;                       // CTA 0: the state snapshot for the scalar tails
};

template <int N, class F>
__device__ __forceinline__ double2 tree2s(const F& leaf, int base = 0) {  // gemv.cu tree2
  if constexpr (N == 1) {
    return leaf(base);
  } else {
    const double2 a = tree2s<N / 2>(leaf, base);
    const double2 b = tree2s<N / 2>(leaf, base + N / 2);
    return make_double2(add(a.x, b.x), add(a.y, b.y));
  }
}

// pairwise over n values v[0..n) (n <= 16) with power-of-two splits; absent past the end
__device__ __forceinline__ double join16(const double* v, int n) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = i < n ? v[i] : 0.0;
#pragma unroll
  for (int h = 1; h < 16; h <<= 1)
#pragma unroll
    for (int i = 0; i + h < 16; i += 2 * h)
      if (i + h < n) x[i] = add(x[i], x[i + h]);
  return x[0];
}

__global__ void __launch_bounds__(SMALL_T, 1) small_iter_kernel(const SmallArgs a) {
  extern __shared__ __align__(128) double ks[];  // this CTA's K tiles [nrb][TILE]
  __shared__ SmallShared sh;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrb = a.nrb, cs = a.cs, n_pad = nrb * TR;
  if (tid == 0) {
    mbar_init(&sh.kbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // K is immutable: its tiles are requested before waiting for the projection (PDL)
  if (tid == 0) {
    mbar_arrive_expect_tx(&sh.kbar, (uint32_t)(nrb * TILE_BYTES));
    for (int rb = 0; rb < nrb; ++rb)
      bulk_g2s(ks + rb * TILE, a.K + tile_offset(rb, rank, a.ncb), TILE_BYTES, &sh.kbar);
  }
  pdl_wait_and_trigger();
  DevState* st = a.st;
  const int status = __ldcg(&st->status);
  mbar_wait(&sh.kbar, 0);  // (no copy outlives the CTA)
  if (status != RUNNING) {  // uniform over the cluster
    cl.sync();
    return;
  }
  const int cur = __ldcg(&st->cur);
  const int64_t c0 = (int64_t)rank * TC;  // this CTA's first column
  if (tid < TC) sh.dv[tid] = __ldcg(a.vb.d + c0 + tid);
  if (rank == 0 && warp == 0) snapshot(&sh.s, st, lane);
  __syncthreads();

  // ---- K d: row t's tile value (fwd_kernel<1>: tree over the 32 column pairs)
  if (tid < n_pad) {
    const int rb = tid >> 5, i = tid & 31;
    const double* kt = ks + rb * TILE;
    sh.kdp[tid] = tree<32>([&](int q) {
      const int o = 64 * q + (i ^ (q & 15));  // in_tile(i, 2q); column 2q + 1 is 32 later
      return add(mul(kt[o], sh.dv[2 * q]), mul(kt[o + 32], sh.dv[2 * q + 1]));
    });
  }
  cl.sync();
  // ---- join the tiles (column order), a = (Kx - y)'Kd and b = ||Kd||^2 per 32-row group
  const double* rcur = a.vb.r[cur];
  if (tid < n_pad) {
    double v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = r < cs ? cl.map_shared_rank(sh.kdp, r)[tid] : 0.0;
    const double kd = join16(v, cs);
    sh.kd[tid] = kd;
    const double l0 = warp_tree(mul(__ldcg(rcur + tid), kd));  // gpss.cpp:195
    const double l1 = warp_tree(mul(kd, kd));                   // gpss.cpp:196
    if (lane == 0) {
      sh.grp[0][warp] = l0;
      sh.grp[1][warp] = l1;
    }
  }
  __syncthreads();
  // ---- backtracking on the exact quadratic (gpss.cpp:199-203), in every CTA alike
  if (tid == 0) {
    const double A = join16(sh.grp[0], nrb), B = join16(sh.grp[1], nrb);
    const int fl = __ldcg(&st->fh_len);
    double f_max = __ldcg(&st->fh[0]);
    for (int i = 1; i < fl; ++i) {
      const double fi = __ldcg(&st->fh[i]);
      f_max = fi > f_max ? fi : f_max;  // as fwd_tail (steps.cuh)
    }
    l1g_gp_config cfg = st->cfg;
    double step = 0.0, f_new = 0.0;
    int h = 0;
    const bool ok = backtrack_quadratic(__ldcg(&st->f), A, B, f_max, __ldcg(&st->gd), cfg,
                                        &step, &f_new, &h);
    sh.lam = step;
    sh.ok = ok;
    if (rank == 0) {  // fwd_tail (steps.cuh), and the same values in the snapshot
      fwd_tail(st, sh.s, FWD_ITER, A, B);
      sh.s.a = A;
      sh.s.b = B;
      sh.s.f_max = f_max;
      sh.s.step = step;
      sh.s.f_new = f_new;
      sh.s.halvings = h;
    }
  }
  __syncthreads();
  if (!sh.ok) {  // backtracking cap: the run failed (fwd_tail set it); uniform
    cl.sync();
    return;
  }
  const double lam = sh.lam;
  // ---- r' = r + lambda K d (gpss.cpp:209)
  if (tid < n_pad) {
    const double rn = add(__ldcg(rcur + tid), mul(lam, sh.kd[tid]));
    sh.rn[tid] = rn;
    if (rank == 0) {
      a.vb.r[cur ^ 1][tid] = rn;
      a.vb.kd[tid] = sh.kd[tid];
    }
  }
  __syncthreads();
  // ---- K^T r': per row tile and column pair, the tile subtree over its 32 rows
  {
    const int q = tid & 31, rb = tid >> 5;  // 32 column pairs x up to 16 row tiles
    if (rb < nrb) {
      const double* kt = ks + rb * TILE;
      const double2 v = tree2s<32>([&](int k) {
        const int o = 64 * q + (k ^ (q & 15));
        const double r = sh.rn[rb * TR + k];
        return make_double2(mul(kt[o], r), mul(kt[o + 32], r));
      });
      sh.colp[rb][2 * q] = v.x;
      sh.colp[rb][2 * q + 1] = v.y;
    }
  }
  __syncthreads();
  // ---- g' = 2 K^T r', x' = x + lambda d, the secant dots (adj_finish)
  if (warp == 0) {
    double t0[16], t1[16];
#pragma unroll
    for (int rb = 0; rb < 16; ++rb) {
      t0[rb] = rb < nrb ? sh.colp[rb][2 * lane] : 0.0;
      t1[rb] = rb < nrb ? sh.colp[rb][2 * lane + 1] : 0.0;
    }
    const double s0 = join16(t0, nrb), s1 = join16(t1, nrb);
    const double g0 = mul(2.0, s0), g1 = mul(2.0, s1);  // gpss.cpp:211
    const int64_t col = c0 + 2 * lane;
    const double2 xo = __ldcg(reinterpret_cast<const double2*>(a.vb.x[cur] + col));
    const double2 go = __ldcg(reinterpret_cast<const double2*>(a.vb.g[cur] + col));
    const double x0n = add(xo.x, mul(lam, sh.dv[2 * lane]));       // gpss.cpp:208
    const double x1n = add(xo.y, mul(lam, sh.dv[2 * lane + 1]));
    *reinterpret_cast<double2*>(a.vb.x[cur ^ 1] + col) = make_double2(x0n, x1n);
    *reinterpret_cast<double2*>(a.vb.g[cur ^ 1] + col) = make_double2(g0, g1);
    const double sa = sub(x0n, xo.x), sb = sub(x1n, xo.y);  // gpss.cpp:150-151
    const double za = sub(g0, go.x), zb = sub(g1, go.y);
    const double dsz = warp_tree(add(mul(sa, za), mul(sb, zb)));
    const double dss = warp_tree(add(mul(sa, sa), mul(sb, sb)));
    const double dzz = warp_tree(add(mul(za, za), mul(zb, zb)));
    if (lane == 0) {
      double* dst = cl.map_shared_rank(&sh.gsum[0][0], 0) + 3 * rank;
      dst[0] = dsz;
      dst[1] = dss;
      dst[2] = dzz;
    }
  }
  cl.sync();
  // ---- the groups pairwise, then the state advance and loop bookkeeping (adj_tail)
  if (rank == 0 && tid == 0) {
    double v[3][16];
    for (int r = 0; r < 16; ++r)
      for (int c = 0; c < 3; ++c) v[c][r] = r < cs ? sh.gsum[r][c] : 0.0;
    adj_tail(st, sh.s, join16(v[0], cs), join16(v[1], cs), join16(v[2], cs));
  }
}

// ---------------------------------------------------------------- host side
bool small_iter_fits(const GemvPlan& pl) {
  return pl.n_pad <= SMALL_MAX_RB * TR && pl.ncb <= SMALL_MAX_CS &&
         (size_t)pl.nrb * TILE_BYTES <= 200 * 1024;
}

void launch_small_iter(const Op& op, const VecBufs* vb, DevState* st, cudaStream_t s) {
  const GemvPlan& pl = op.plan;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(small_iter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SMALL_MAX_RB * TILE_BYTES));
    L1G_CUDA(cudaFuncSetAttribute(small_iter_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  SmallArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.nrb = (int)pl.nrb;
  a.cs = (int)pl.ncb;
  a.st = st;
  a.vb = *vb;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.cs, 1, 1);
  cfg.blockDim = dim3(SMALL_T, 1, 1);
  cfg.dynamicSmemBytes = (size_t)a.nrb * TILE_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = (unsigned)a.cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  L1G_CUDA(cudaLaunchKernelEx(&cfg, small_iter_kernel, a));
}

}  // namespace l1g
