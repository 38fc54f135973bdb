// gemv.cu -- fused fp64 forward (K d) and adjoint (K^T r) products over the tiled K.
//
// Replaces DenseOperator::do_apply / do_apply_adjoint (linear_operator.hpp:45-48) on the
// GPSS hot path (gpss.cpp:194-196 and :206-211).  Both kernels are persistent (one CTA per
// SM) and warp specialised: warp 0 streams 32x64 K tiles into a 3-stage shared-memory ring
// with cp.async.bulk (TMA engine) + mbarriers; warps 1-4 reduce them.  Every output is the
// canonical pairwise sum of rounded products (common.cuh), evaluated as
//   per-lane 32/64-leaf trees inside a tile -> a binary counter over the tiles of a task ->
//   a tree over task partials, done by the CTA that completes a group last.
// The same completing CTA runs the fused epilogue:
//   forward/ITER : a = (Kx - y)'Kd, b = ||Kd||^2, then the backtracking line search;
//   forward/INIT : r = Kx0 - y, f = ||r||^2;
//   adjoint/ITER : r += lambda Kd (prologue), g' = 2 K^T r, x' = x + lambda d,
//                  s'z, s's, z'z for the next BB step, telemetry, stop tests.
#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"

namespace l1g {

constexpr int NCONS = 4;                 // consumer warps
constexpr int NTHREADS = 32 * (NCONS + 1);
constexpr int STAGES = 3;
constexpr int FWD_STAGE_DBL = 4 * TILE + 64;   // 4 tiles + the matching 64-entry slice of d
constexpr int ADJ_STAGE_DBL = 4 * TILE;
constexpr int FWD_MAX_STAGES = 128;      // column blocks per forward task (counter depth 8)
constexpr int ADJ_MAX_BLOCKS = 32;       // row blocks per adjoint task (counter depth 6)
constexpr int MAX_TR = ADJ_MAX_BLOCKS * TR;

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
  DevState* st;
  VecBufs vb;
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

// Tree over `count` values v[0..count) (runtime count, absent beyond) by one warp: lane l
// takes block l of each 32-chunk, the butterfly reduces the chunk, a counter joins chunks.
__device__ __forceinline__ double warp_tree_array(const double* v, int count, int stride,
                                                  int lane) {
  Counter<20> acc;
  const int chunks = (count + 31) >> 5;
  for (int c = 0; c < chunks; ++c) {
    const int i = c * 32 + lane;
    double x = i < count ? __ldcg(v + (int64_t)i * stride) : 0.0;
    x = warp_tree(x);
    acc.push(x, c);
  }
  return acc.final_value(chunks);
}

// ============================================================================ forward
__device__ __noinline__ void fwd_finish(const FwdArgs& a, int rg, int ct, int cw, int lane,
                                        double (*wsum)[3], int* s_flag) {
  const int64_t row = (int64_t)rg * ROW_GROUP + ct;
  Counter<20> acc;
  for (int cr = 0; cr < a.ncr; ++cr) acc.push(__ldcg(a.part + (int64_t)cr * a.n_pad + row), cr);
  const double kd = acc.final_value(a.ncr);
  if (a.mode == FWD_APPLY) {
    a.vout[row] = kd;
    if (ct == 0) a.cnt_grp[rg] = 0;
    return;
  }
  const int cur = a.st->cur;
  double l0, l1 = 0.0;
  if (a.mode == FWD_INIT) {
    const double r = sub(kd, a.vb.y[row]);  // Kx0 - y   (gpss.cpp:128)
    a.vb.r[cur][row] = r;
    l0 = mul(r, r);                         // ||r||^2   (gpss.cpp:129)
  } else {
    a.vb.kd[row] = kd;
    l0 = mul(a.vb.r[cur][row], kd);         // (Kx-y)'Kd (gpss.cpp:195)
    l1 = mul(kd, kd);                       // ||Kd||^2  (gpss.cpp:196)
  }
  l0 = warp_tree(l0);
  l1 = warp_tree(l1);
  if (lane == 0) {
    wsum[cw][0] = l0;
    wsum[cw][1] = l1;
  }
  named_bar_sync(1, 32 * NCONS);
  if (ct == 0) {
    a.grpsum[2 * rg + 0] = add(add(wsum[0][0], wsum[1][0]), add(wsum[2][0], wsum[3][0]));
    a.grpsum[2 * rg + 1] = add(add(wsum[0][1], wsum[1][1]), add(wsum[2][1], wsum[3][1]));
    a.cnt_grp[rg] = 0;
    __threadfence();
    const unsigned old = atomicAdd(a.cnt_all, 1u);
    *s_flag = (old == (unsigned)a.nrg - 1u);
  }
  named_bar_sync(1, 32 * NCONS);
  if (!*s_flag) return;
  __threadfence();
  if (cw != 0) return;
  const double A = warp_tree_array(a.grpsum + 0, a.nrg, 2, lane);
  const double B = warp_tree_array(a.grpsum + 1, a.nrg, 2, lane);
  if (lane != 0) return;
  DevState* st = a.st;
  *a.cnt_all = 0;
  if (a.mode == FWD_INIT) {
    st->f = A;
    st->f_prev = A;
    st->fh[0] = A;
    st->fh_len = 1;
    return;
  }
  // gpss.cpp:199-203 -- nonmonotone reference value and quadratic backtracking
  st->a = A;
  st->b = B;
  double f_max = st->fh[0];
  for (int i = 1; i < st->fh_len; ++i) f_max = st->fh[i] > f_max ? st->fh[i] : f_max;
  st->f_max = f_max;
  double step, f_new;
  int h;
  if (backtrack_quadratic(st->f, A, B, f_max, st->gd, st->cfg, &step, &f_new, &h)) {
    st->step = step;
    st->f_new = f_new;
    st->halvings = h;
  } else {
    st->status = FAILED;
    st->failure = FAIL_BACKTRACK;
  }
}

__global__ void __launch_bounds__(NTHREADS, 1) fwd_kernel(const FwdArgs a) {
  if (a.mode != FWD_APPLY && a.st->status != RUNNING) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sbase = reinterpret_cast<double*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * FWD_STAGE_DBL * 8);
  uint64_t* empty = full + STAGES;
  __shared__ double wsum[NCONS][3];
  __shared__ int s_last, s_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
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
          mbar_arrive_expect_tx(&full[stage], 4 * TILE_BYTES + 512);
#pragma unroll
          for (int w = 0; w < 4; ++w)
            bulk_g2s(dst + w * TILE, a.K + tile_offset(4 * rg + w, cb0 + s, a.ncb), TILE_BYTES,
                     &full[stage]);
          bulk_g2s(dst + 4 * TILE, a.vin + (cb0 + s) * TC, 512, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  // ---- consumers: warp cw owns row block 4*rg + cw, lane = row inside the block
  const int cw = warp - 1, ct = threadIdx.x - 32;
  const int sw = lane & 7;
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
      const double2* ku = reinterpret_cast<const double2*>(sb + cw * TILE) + lane * 32;
      const double2* du = reinterpret_cast<const double2*>(sb + 4 * TILE);
      const double v = tree<32>([&](int q) {
        const double2 k = ku[q ^ sw];
        const double2 d = du[q];
        return add(mul(k.x, d.x), mul(k.y, d.y));
      });
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      acc.push(v, (uint32_t)s);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    const int64_t row = (int64_t)rg * ROW_GROUP + ct;
    a.part[(int64_t)cr * a.n_pad + row] = acc.final_value((uint32_t)nst);
    __threadfence();
    named_bar_sync(1, 32 * NCONS);
    if (ct == 0) {
      const unsigned old = atomicAdd(&a.cnt_grp[rg], 1u);
      s_last = (old == (unsigned)a.ncr - 1u);
    }
    named_bar_sync(1, 32 * NCONS);
    if (s_last) {
      __threadfence();
      fwd_finish(a, rg, ct, cw, lane, wsum, &s_flag);
    }
    named_bar_sync(1, 32 * NCONS);
  }
}

// ============================================================================ adjoint
__device__ __noinline__ void adj_finish(const AdjArgs& a, int cg, int ct, int cw, int lane,
                                        double (*wsum)[3], int* s_flag) {
  const int64_t col = (int64_t)cg * COL_GROUP + 2 * ct;
  Counter<20> acc0, acc1;
  for (int rr = 0; rr < a.nrr; ++rr) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(a.part + (int64_t)rr * a.p_pad + col));
    acc0.push(v.x, rr);
    acc1.push(v.y, rr);
  }
  const double s0 = acc0.final_value(a.nrr), s1 = acc1.final_value(a.nrr);
  if (a.mode == ADJ_APPLY) {
    *reinterpret_cast<double2*>(a.vout + col) = make_double2(s0, s1);
    if (ct == 0) a.cnt_grp[cg] = 0;
    return;
  }
  DevState* st = a.st;
  const int cur = st->cur;
  const double g0 = mul(2.0, s0), g1 = mul(2.0, s1);  // 2 K^T r (gpss.cpp:130, :211)
  if (a.mode == ADJ_INIT) {
    *reinterpret_cast<double2*>(a.vb.g[cur] + col) = make_double2(g0, g1);
    if (ct == 0) a.cnt_grp[cg] = 0;
    return;
  }
  // ADJ_ITER epilogue: x' = x + lambda d (gpss.cpp:208), s = x' - x, z = g' - g (:150-151)
  const double lam = st->step;
  const double2 xo = *reinterpret_cast<const double2*>(a.vb.x[cur] + col);
  const double2 go = *reinterpret_cast<const double2*>(a.vb.g[cur] + col);
  const double2 dd = *reinterpret_cast<const double2*>(a.vb.d + col);
  const double x0n = add(xo.x, mul(lam, dd.x)), x1n = add(xo.y, mul(lam, dd.y));
  *reinterpret_cast<double2*>(a.vb.x[cur ^ 1] + col) = make_double2(x0n, x1n);
  *reinterpret_cast<double2*>(a.vb.g[cur ^ 1] + col) = make_double2(g0, g1);
  const double sa = sub(x0n, xo.x), sb = sub(x1n, xo.y);
  const double za = sub(g0, go.x), zb = sub(g1, go.y);
  double lsz = add(mul(sa, za), mul(sb, zb));
  double lss = add(mul(sa, sa), mul(sb, sb));
  double lzz = add(mul(za, za), mul(zb, zb));
  lsz = warp_tree(lsz);
  lss = warp_tree(lss);
  lzz = warp_tree(lzz);
  if (lane == 0) {
    wsum[cw][0] = lsz;
    wsum[cw][1] = lss;
    wsum[cw][2] = lzz;
  }
  named_bar_sync(1, 32 * NCONS);
  if (ct == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      a.grpsum[3 * cg + c] = add(add(wsum[0][c], wsum[1][c]), add(wsum[2][c], wsum[3][c]));
    a.cnt_grp[cg] = 0;
    __threadfence();
    const unsigned old = atomicAdd(a.cnt_all, 1u);
    *s_flag = (old == (unsigned)a.ncg - 1u);
  }
  named_bar_sync(1, 32 * NCONS);
  if (!*s_flag) return;
  __threadfence();
  if (cw != 0) return;
  const double SZ = warp_tree_array(a.grpsum + 0, a.ncg, 3, lane);
  const double SS = warp_tree_array(a.grpsum + 1, a.ncg, 3, lane);
  const double ZZ = warp_tree_array(a.grpsum + 2, a.ncg, 3, lane);
  if (lane != 0) return;
  *a.cnt_all = 0;
  // gpss.cpp:206-217 state advance, gpss.cpp:255-283 loop bookkeeping
  st->sz = SZ;
  st->ss = SS;
  st->zz = ZZ;
  st->f = st->f_new;
  if (st->fh_len < kMaxHist) {
    st->fh[st->fh_len++] = st->f;
  } else {
    for (int i = 0; i + 1 < st->fh_len; ++i) st->fh[i] = st->fh[i + 1];
    st->fh[st->fh_len - 1] = st->f;
  }
  while (st->fh_len > st->cfg.memory) {
    for (int i = 0; i + 1 < st->fh_len; ++i) st->fh[i] = st->fh[i + 1];
    --st->fh_len;
  }
  const int64_t k = st->k;
  st->k = k + 1;
  st->matvecs += 2;
  l1g_iter_record rec;
  rec.k = k;
  rec.f = st->f;
  rec.stationarity = st->stat;
  rec.alpha = st->alpha_used;
  rec.step = st->step;
  rec.matvecs = st->matvecs;
  rec.elapsed_seconds = elapsed_s(st);
  rec.bb_active = st->choice.bb_active;
  rec.halvings = st->halvings;
  rec.bb1_raw = st->choice.bb1_raw;
  rec.bb2_raw = st->choice.bb2_raw;
  rec.tau_before = st->choice.tau_before;
  rec.tau_after = st->choice.tau_after;
  rec.f_max = st->f_max;
  rec.dir_derivative = st->gd;
  rec.theta = st->theta;
  rec.support = st->support;
  st->last = rec;
  if (st->trace && k < st->trace_cap) st->trace[k] = rec;
  if (!st->single_step && st->objective_tol > 0.0) {
    const double af = fabs(st->f);
    if (fabs(sub(st->f_prev, st->f)) <= mul(st->objective_tol, af > 1.0 ? af : 1.0)) {
      st->status = STOPPED;
      st->reason = L1G_OBJECTIVE_TOL;
    }
  }
  st->f_prev = st->f;
  st->cur = cur ^ 1;
}

__global__ void __launch_bounds__(NTHREADS, 1) adj_kernel(const AdjArgs a) {
  if (a.mode != ADJ_APPLY && a.st->status != RUNNING) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sbase = reinterpret_cast<double*>(smem);
  double* rs = sbase + (size_t)STAGES * ADJ_STAGE_DBL;
  uint64_t* full = reinterpret_cast<uint64_t*>(rs + MAX_TR);
  uint64_t* empty = full + STAGES;
  __shared__ double wsum[NCONS][3];
  __shared__ int s_last, s_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int ntasks = a.ncg * a.nrr;
  const int64_t tr = (int64_t)a.blocks * TR;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int cg = t / a.nrr, rr = t - cg * a.nrr;
        const int64_t rb0 = (int64_t)rr * a.blocks;
        const int nb = (int)(a.nrb - rb0 < (int64_t)a.blocks ? a.nrb - rb0 : (int64_t)a.blocks);
        for (int s = 0; s < nb; ++s) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&full[stage], 4 * TILE_BYTES);
          bulk_g2s(sbase + (size_t)stage * ADJ_STAGE_DBL,
                   a.K + tile_offset(rb0 + s, 4 * (int64_t)cg, a.ncb), 4 * TILE_BYTES,
                   &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }
  const int cw = warp - 1, ct = threadIdx.x - 32;
  const int cur = (a.mode == ADJ_APPLY) ? 0 : a.st->cur;
  const double lam = (a.mode == ADJ_ITER) ? a.st->step : 0.0;
  const double* rin = (a.mode == ADJ_APPLY) ? a.vin : a.vb.r[cur];
  int stage = 0;
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const int cg = t / a.nrr, rr = t - cg * a.nrr;
    const int64_t rb0 = (int64_t)rr * a.blocks;
    const int nb = (int)(a.nrb - rb0 < (int64_t)a.blocks ? a.nrb - rb0 : (int64_t)a.blocks);
    const int64_t row0 = rr * tr;
    // prologue: the task's slice of r (ITER: r + lambda Kd, gpss.cpp:209)
    for (int i = ct; i < nb * TR; i += 32 * NCONS) {
      double r = rin[row0 + i];
      if (a.mode == ADJ_ITER) {
        r = add(r, mul(lam, a.vb.kd[row0 + i]));
        if (cg == 0) a.vb.r[cur ^ 1][row0 + i] = r;
      }
      rs[i] = r;
    }
    named_bar_sync(1, 32 * NCONS);
    Counter<6> acc0, acc1;
    for (int s = 0; s < nb; ++s) {
      mbar_wait(&full[stage], phase);
      const double2* ku =
          reinterpret_cast<const double2*>(sbase + (size_t)stage * ADJ_STAGE_DBL + cw * TILE);
      const double* rr_s = rs + s * TR;
      const double2 v = tree2<32>([&](int i) {
        const double2 k = ku[i * 32 + (lane ^ (i & 7))];
        const double r = rr_s[i];
        return make_double2(mul(k.x, r), mul(k.y, r));
      });
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      acc0.push(v.x, (uint32_t)s);
      acc1.push(v.y, (uint32_t)s);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    const int64_t col = (int64_t)cg * COL_GROUP + cw * TC + 2 * lane;
    *reinterpret_cast<double2*>(a.part + (int64_t)rr * a.p_pad + col) =
        make_double2(acc0.final_value((uint32_t)nb), acc1.final_value((uint32_t)nb));
    __threadfence();
    named_bar_sync(1, 32 * NCONS);
    if (ct == 0) {
      const unsigned old = atomicAdd(&a.cnt_grp[cg], 1u);
      s_last = (old == (unsigned)a.nrr - 1u);
    }
    named_bar_sync(1, 32 * NCONS);
    if (s_last) {
      __threadfence();
      adj_finish(a, cg, ct, cw, lane, wsum, &s_flag);
    }
    named_bar_sync(1, 32 * NCONS);
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
  pl.grid = sm_count;
  return pl;
}

static size_t fwd_smem() { return (size_t)STAGES * FWD_STAGE_DBL * 8 + 2 * STAGES * 8; }
static size_t adj_smem() { return (size_t)STAGES * ADJ_STAGE_DBL * 8 + MAX_TR * 8 + 2 * STAGES * 8; }

void launch_fwd(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout, const VecBufs* vb,
                DevState* st, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    L1G_CUDA(cudaFuncSetAttribute(fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)fwd_smem()));
    attr = true;
  }
  const GemvPlan& pl = op.plan;
  FwdArgs a{};
  a.K = op.K;
  a.ncb = pl.ncb;
  a.n_pad = pl.n_pad;
  a.stages = pl.fwd_stages;
  a.nrg = pl.nrg;
  a.ncr = pl.ncr;
  a.mode = mode;
  a.vin = (mode == FWD_ITER) ? vb->d : vin;
  a.vout = vout;
  a.part = ws.fwd_part;
  a.grpsum = ws.grpsum;
  a.cnt_grp = ws.counters;
  a.cnt_all = ws.counters + pl.nrg + pl.ncg;
  a.st = st;
  if (vb) a.vb = *vb;
  const int grid = (int)std::min<int64_t>(pl.grid, (int64_t)pl.nrg * pl.ncr);
  fwd_kernel<<<grid, NTHREADS, fwd_smem(), s>>>(a);
  L1G_CUDA(cudaGetLastError());
}

void launch_adj(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout, const VecBufs* vb,
                DevState* st, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    L1G_CUDA(cudaFuncSetAttribute(adj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)adj_smem()));
    attr = true;
  }
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
  const int grid = (int)std::min<int64_t>(pl.grid, (int64_t)pl.ncg * pl.nrr);
  adj_kernel<<<grid, NTHREADS, adj_smem(), s>>>(a);
  L1G_CUDA(cudaGetLastError());
}

}  // namespace l1g
