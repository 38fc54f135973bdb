// project.cu -- Euclidean projection onto the l1 ball as one thread-block cluster.
//
// Replaces project_l1_ball_with_threshold (prox.cpp:38-73) and, in PROJ_ITER mode, steps
// 1-3 of gp_iterate (gpss.cpp:146-192): steplength choice, v = x - alpha g, h = P(v),
// d = h - x, ||h - x||_inf, g'd and the alpha escalation loop, all on device.
//
// A cluster of `cs` CTAs keeps v resident in distributed shared memory (CTA r owns the
// aligned slice [r*ls, (r+1)*ls)).  The threshold is found without a host sort:
//   1. Michelot's pivot iteration (cluster-wide counts and sums) brackets theta;
//   2. the elements above the bracket (plus the largest one below it) are gathered into
//      CTA 0 and bitonic-sorted (shared memory, or L2-resident global memory if large);
//   3. one thread forms the *sequential* descending prefix sums exactly as prox.cpp:43-52
//      does, then all threads test |v|_(k) > (S_k - rho)/k in parallel and the first
//      failure fixes theta -- bit-identical to the reference's sort-and-scan;
//   4. the feasibility bump loop of prox.cpp:58-65 on canonical cluster-wide l1 norms.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"

namespace cg = cooperative_groups;

namespace l1g {

constexpr int PT = 512;
constexpr int PW = PT / 32;
constexpr int64_t MAX_LS = 16384;
constexpr int MAX_CS = 16;

struct ProjArgs {
  int mode;
  int64_t p, p_pad, ls;
  int cs;
  int64_t cand_cap;
  const double* xin;
  const double* gin;
  double* out;
  double* gcand;  // global scratch: candidates (next_pow2(p_pad) + 1)
  double* gpre;   // global scratch: sequential prefix sums (p_pad + 2)
  DevState* st;
  VecBufs vb;
};

struct ProjShared {
  double slot[2][MAX_CS][4];  // cluster reduction slots (double-buffered)
  double wv[PW][4];
  double bc[8];
  long long wl[PW][2];
  long long slotl[2][MAX_CS][2];
  int red_par;
};

// ---------------------------------------------------------------- block helpers
// canonical tree over the CTA slice: warp w owns contiguous 32-element chunks
template <class F>
__device__ __forceinline__ double slice_tree(int64_t ls, const F& leaf, ProjShared& sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = ls >> 5;
  const int64_t per = nchunks >= PW ? nchunks / PW : 1;
  const int active = nchunks >= PW ? PW : (int)nchunks;
  double v = 0.0;
  if (warp < active) {
    Counter<16> acc;
    for (int64_t c = 0; c < per; ++c) {
      const int64_t j = ((int64_t)warp * per + c) * 32 + lane;
      acc.push(warp_tree(leaf(j)), (uint32_t)c);
    }
    v = acc.final_value((uint32_t)per);
  }
  if (lane == 0) sh.wv[warp][0] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    double x = lane < PW ? sh.wv[lane][0] : 0.0;
#pragma unroll
    for (int o = 1; o < PW; o <<= 1) x = add(x, __shfl_xor_sync(0xffffffffu, x, o));
    r = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) sh.wv[0][1] = r;
  __syncthreads();
  r = sh.wv[0][1];
  __syncthreads();
  return r;
}

// Cluster-wide combine of per-CTA values.  kinds[c]: 0 = canonical tree sum over ranks,
// 1 = max, 2 = plain sum.  Every CTA of the cluster must call it in the same order.
__device__ void cluster_combine(double* vals, const int* kinds, int nv, ProjShared& sh,
                                cg::cluster_group& cl, int cs) {
  const int par = sh.red_par;
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0)
    for (int c = 0; c < nv; ++c) sh.slot[par][rank][c] = vals[c];
  cl.sync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int c = 0; c < nv; ++c) {
      double x = 0.0;
      if (lane < cs) {
        const ProjShared* rem = cl.map_shared_rank(&sh, lane);
        x = rem->slot[par][lane][c];
      }
      for (int o = 1; o < cs; o <<= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, x, o);
        x = kinds[c] == 1 ? fmax(x, y) : add(x, y);
      }
      if (lane == 0) sh.bc[c] = x;
    }
  }
  __syncthreads();
  for (int c = 0; c < nv; ++c) vals[c] = sh.bc[c];
  __syncthreads();
  if (threadIdx.x == 0) sh.red_par = par ^ 1;
  __syncthreads();
}

__device__ __forceinline__ double block_max(double v, ProjShared& sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_max(v);
  if (lane == 0) sh.wv[warp][2] = v;
  __syncthreads();
  if (warp == 0) {
    double x = lane < PW ? sh.wv[lane][2] : -1.0;
    x = warp_max(x);
    if (lane == 0) sh.wv[0][3] = x;
  }
  __syncthreads();
  const double r = sh.wv[0][3];
  __syncthreads();
  return r;
}

__device__ __forceinline__ long long block_sum_ll(long long v, ProjShared& sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum_ll(v);
  if (lane == 0) sh.wl[warp][0] = v;
  __syncthreads();
  long long r = 0;
  for (int w = 0; w < PW; ++w) r += sh.wl[w][0];
  __syncthreads();
  return r;
}

// exclusive prefix of per-thread counts inside the block
__device__ __forceinline__ long long block_excl_scan(long long v, ProjShared& sh,
                                                     long long* total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh.wl[warp][1] = inc;
  __syncthreads();
  long long base = 0, tot = 0;
  for (int w = 0; w < PW; ++w) {
    if (w < warp) base += sh.wl[w][1];
    tot += sh.wl[w][1];
  }
  __syncthreads();
  *total = tot;
  return base + inc - v;
}

template <class T>
__device__ void bitonic_desc(T* c, int64_t n2) {
  for (int64_t k = 2; k <= n2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < n2; i += PT) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const double a = c[i], b = c[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) {
            c[i] = b;
            c[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(PT, 1) proj_kernel(const ProjArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int cs = a.cs;
  extern __shared__ __align__(16) double dyn[];
  double* vs = dyn;               // v slice (ls)
  double* cand = dyn + a.ls;      // CTA 0 candidate buffer (cand_cap + 1)
  __shared__ ProjShared sh;
  __shared__ int s_dec;
  DevState* st = a.st;
  if (threadIdx.x == 0) sh.red_par = 0;
  const bool prof = (a.mode == PROJ_ITER) && cl.block_rank() == 0 && threadIdx.x == 0;
  long long t_last = clock64();
  auto mark = [&](int idx) {
    if (prof) {
      const long long t = clock64();
      st->prof[idx] += (double)(t - t_last);
      t_last = t;
    }
  };
  auto count = [&](int idx, double v) {
    if (prof) st->prof[idx] += v;
  };
  if (a.mode == PROJ_ITER && st->status != RUNNING) return;  // uniform over the cluster
  const l1g_gp_config cfg = st->cfg;
  const double rho = a.mode == PROJ_PLAIN ? st->rho : st->rho;
  const int cur = a.mode == PROJ_ITER ? st->cur : 0;
  const double* x = a.mode == PROJ_ITER ? a.vb.x[cur] : a.xin;
  const double* g = a.mode == PROJ_ITER ? a.vb.g[cur] : a.gin;
  const int64_t base = (int64_t)rank * a.ls;
  const int64_t lim = a.p_pad - base < a.ls ? (a.p_pad - base > 0 ? a.p_pad - base : 0) : a.ls;

  // ---- steplength and loop-top checks (gpss.cpp:233-245, :147-153), CTA 0 decides
  double alpha = 1.0, first_alpha = 1.0;
  if (a.mode == PROJ_ITER) {
    if (rank == 0 && threadIdx.x == 0) {
      int dec = 0;
      if (!st->single_step) {
        if (st->max_iterations > 0 && st->k >= st->max_iterations) dec = 1 + L1G_MAX_ITERATIONS;
        else if (st->max_matvecs > 0 && st->matvecs >= st->max_matvecs) dec = 1 + L1G_MAX_MATVECS;
        else if (st->max_seconds > 0.0 && elapsed_s(st) >= st->max_seconds) dec = 1 + L1G_MAX_SECONDS;
      } else if (st->stationary) {
        dec = 1 + L1G_STATIONARY;
      }
      double al = st->alpha0;
      if (dec == 0) {
        if (st->k == 0) {
          l1g_sl_choice c;
          c.alpha = st->alpha0;
          c.bb_active = 0;
          c.bb1_raw = c.bb2_raw = c.tau_before = c.tau_after = nan_d();
          st->choice = c;
        } else {
          steplength_from_dots(&st->tau, st->a2h, &st->a2_len, st->sz, st->ss, st->zz, cfg,
                               &st->choice);
        }
        al = st->choice.alpha;
      } else {
        st->status = STOPPED;
        st->reason = dec - 1;
        if (dec - 1 == L1G_STATIONARY) {
          st->last.stationarity = 0.0;
          st->out_stationarity = 0.0;
        }
      }
      sh.bc[6] = al;
      s_dec = dec;
    }
    cl.sync();
    if (threadIdx.x == 0) {
      const ProjShared* r0 = cl.map_shared_rank(&sh, 0);
      const int* d0 = cl.map_shared_rank(&s_dec, 0);
      sh.bc[7] = r0->bc[6];
      s_dec = *d0;
    }
    cl.sync();
    if (s_dec != 0) return;
    alpha = first_alpha = sh.bc[7];
  }

  double first_stat = 0.0;
  count(8, 1.0);
  mark(0);
  for (int attempt = 0;; ++attempt) {
    count(9, 1.0);
    // ---- v = x - alpha g  (gpss.cpp:167; alpha0: x0 - grad, gpss.cpp:95)
    for (int64_t j = threadIdx.x; j < a.ls; j += PT) {
      double v = 0.0;
      if (j < lim) {
        const int64_t gj = base + j;
        if (a.mode == PROJ_PLAIN) v = x[gj];
        else if (a.mode == PROJ_ALPHA0) v = sub(x[gj], g[gj]);
        else v = sub(x[gj], mul(alpha, g[gj]));
      }
      vs[j] = v;
    }
    __syncthreads();
    double red[4];
    const int k_l1max[2] = {0, 1};
    red[0] = slice_tree(a.ls, [&](int64_t j) { return fabs(vs[j]); }, sh);
    double lm = 0.0;
    for (int64_t j = threadIdx.x; j < a.ls; j += PT) lm = fmax(lm, fabs(vs[j]));
    red[1] = block_max(lm, sh);
    cluster_combine(red, k_l1max, 2, sh, cl, cs);
    const double l1v = red[0], vinf = red[1];
    mark(1);

    // ---- threshold (prox.cpp:40-53)
    double theta = 0.0;
    int branch;  // 0: rho == 0, 1: already feasible, 2: threshold
    if (rho == 0.0) {
      branch = 0;
      theta = vinf;
    } else if (l1v <= rho) {
      branch = 1;
    } else {
      branch = 2;
      // Michelot pivot iteration: theta_{t+1} = (sum_{|v|>theta_t} |v| - rho) / #{|v|>theta_t}
      double th = dvd(sub(l1v, rho), (double)a.p_pad);
      double cnt_prev = -1.0;
      const int kinds_cs[2] = {2, 2};
      for (int it = 0; it < 64; ++it) {
        double c = 0.0, s = 0.0;
        for (int64_t j = threadIdx.x; j < lim; j += PT) {
          const double m = fabs(vs[j]);
          if (m > th) {
            c += 1.0;
            s += m;
          }
        }
        // block sums (order irrelevant: only brackets the exact search below)
        c = warp_tree(c);
        s = warp_tree(s);
        if ((threadIdx.x & 31) == 0) {
          sh.wv[threadIdx.x >> 5][0] = c;
          sh.wv[threadIdx.x >> 5][1] = s;
        }
        __syncthreads();
        double cc = 0.0, ss = 0.0;
        for (int w = 0; w < PW; ++w) {
          cc += sh.wv[w][0];
          ss += sh.wv[w][1];
        }
        __syncthreads();
        double v2[2] = {cc, ss};
        cluster_combine(v2, kinds_cs, 2, sh, cl, cs);
        count(10, 1.0);
        if (v2[0] == cnt_prev || v2[0] == 0.0) break;
        cnt_prev = v2[0];
        th = dvd(sub(v2[1], rho), v2[0]);
      }
      mark(2);
      // exact sort-and-scan on the elements above a bracket below theta
      double lo = th > 0.0 ? sub(th, mul(th, 0x1.0p-20)) : -1.0;
      for (int tries = 0;; ++tries) {
        long long myc = 0;
        double mynext = -1.0;
        for (int64_t j = threadIdx.x; j < lim; j += PT) {
          const double m = fabs(vs[j]);
          if (m > lo) ++myc;
          else mynext = fmax(mynext, m);
        }
        long long ctot;
        const long long off = block_excl_scan(myc, sh, &ctot);
        const double bnext = block_max(mynext, sh);
        // cluster: per-rank counts -> offsets; global next
        if (threadIdx.x == 0) {
          sh.slotl[sh.red_par][rank][0] = ctot;
          sh.slot[sh.red_par][rank][0] = bnext;
        }
        cl.sync();
        if (threadIdx.x == 0) {
          long long before = 0, total = 0;
          double nx = -1.0;
          const int par = sh.red_par;
          for (int r = 0; r < cs; ++r) {
            const ProjShared* rem = cl.map_shared_rank(&sh, r);
            const long long cr = rem->slotl[par][r][0];
            if (r < (int)rank) before += cr;
            total += cr;
            nx = fmax(nx, rem->slot[par][r][0]);
          }
          sh.wl[0][0] = before;
          sh.wl[0][1] = total;
          sh.bc[5] = nx;
        }
        __syncthreads();
        const long long before = sh.wl[0][0], total = sh.wl[0][1];
        const double next = sh.bc[5];
        __syncthreads();
        if (threadIdx.x == 0) sh.red_par ^= 1;
        __syncthreads();
        const long long L = total + (next >= 0.0 ? 1 : 0);
        int64_t n2 = 1;
        while (n2 < total) n2 <<= 1;
        const bool in_smem = (n2 + 1 <= a.cand_cap);
        double* cbuf = in_smem ? cl.map_shared_rank(cand, 0) : a.gcand;
        // scatter candidates (order is irrelevant: they are sorted next)
        long long pos = before + off;
        for (int64_t j = threadIdx.x; j < lim; j += PT) {
          const double m = fabs(vs[j]);
          if (m > lo) cbuf[pos++] = m;
        }
        __threadfence();
        cl.sync();
        mark(3);
        count(11, (double)total);
        __shared__ int s_ff;
        if (rank == 0) {
          double* c = in_smem ? cand : a.gcand;
          for (int64_t i = total + threadIdx.x; i < n2; i += PT) c[i] = 0.0;
          __syncthreads();
          bitonic_desc(c, n2);
          if (threadIdx.x == 0 && next >= 0.0) c[total] = next;
          __syncthreads();
          mark(4);
          double* pre = a.gpre;
          if (threadIdx.x == 0) {  // the reference's sequential cumulative sum
            double S = 0.0;
            for (long long i = 0; i < L; ++i) {
              S = add(S, c[i]);
              pre[i] = S;
            }
          }
          __syncthreads();
          long long ff = L;  // first failing index
          for (long long i = threadIdx.x; i < L; i += PT) {
            const double cand_i = dvd(sub(__ldcg(pre + i), rho), (double)(i + 1));
            if (!(c[i] > cand_i)) {
              ff = i;
              break;
            }
          }
          // block min
          ff = -ff;
          {
            long long v = ff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
            if ((threadIdx.x & 31) == 0) sh.wl[threadIdx.x >> 5][0] = v;
            __syncthreads();
            long long m = LLONG_MIN;
            for (int w = 0; w < PW; ++w) m = max(m, sh.wl[w][0]);
            __syncthreads();
            ff = -m;
          }
          if (threadIdx.x == 0) {
            double thv = 0.0;
            if (ff > 0) thv = dvd(sub(__ldcg(pre + ff - 1), rho), (double)ff);
            // all passed although smaller elements exist: the bracket was too high
            const int retry = (ff == L && next >= 0.0) ? 1 : 0;
            sh.bc[4] = thv;
            s_ff = retry;
          }
        }
        cl.sync();
        if (threadIdx.x == 0) {
          const ProjShared* r0 = cl.map_shared_rank(&sh, 0);
          const int* f0 = cl.map_shared_rank(&s_ff, 0);
          sh.bc[3] = r0->bc[4];
          s_dec = *f0;
        }
        cl.sync();
        mark(5);
        if (!s_dec) {
          theta = sh.bc[3];
          break;
        }
        count(13, 1.0);
        lo = (lo > 0.0 && tries < 4) ? mul(lo, 0.5) : -1.0;
      }
      if (theta < 0.0) theta = 0.0;
      // feasibility bump (prox.cpp:58-65)
      double bump = mul(theta > vinf ? theta : vinf, DBL_EPSILON);
      const int k_sum[1] = {0};
      int guard = 0;
      for (;;) {
        double l1u[1];
        const double thc = theta;
        l1u[0] = slice_tree(a.ls, [&](int64_t j) {
          const double v = vs[j];
          return fabs(v > thc ? sub(v, thc) : (v < -thc ? add(v, thc) : 0.0));
        }, sh);
        cluster_combine(l1u, k_sum, 1, sh, cl, cs);
        if (!(l1u[0] > rho && guard++ < 64)) break;
        count(12, 1.0);
        theta = add(theta, bump);
        bump = mul(bump, 2.0);
      }
      mark(6);
    }

    // ---- h, d = h - x, ||h - x||_inf, g'd, support  (gpss.cpp:167-178)
    const double th = theta;
    auto hval = [&](double v) {
      if (branch == 0) return 0.0;
      if (branch == 1) return v;
      return v > th ? sub(v, th) : (v < -th ? add(v, th) : 0.0);
    };
    double lmax = 0.0, hmax = 0.0;
    long long sup = 0;
    for (int64_t j = threadIdx.x; j < a.ls; j += PT) {
      const double h = hval(vs[j]);
      sup += (h != 0.0);
      hmax = fmax(hmax, fabs(h));
      if (j < lim && a.mode != PROJ_ALPHA0) {
        const int64_t gj = base + j;
        const double dj = a.mode == PROJ_PLAIN ? h : sub(h, x[gj]);
        lmax = fmax(lmax, fabs(dj));
        a.out[gj] = dj;
      }
    }
    double gdl = 0.0;
    if (a.mode == PROJ_ITER) {
      gdl = slice_tree(a.ls, [&](int64_t j) {
        if (j >= lim) return 0.0;
        const int64_t gj = base + j;
        return mul(g[gj], sub(hval(vs[j]), x[gj]));
      }, sh);
    }
    double red2[4] = {gdl, block_max(lmax, sh), block_max(hmax, sh),
                      (double)block_sum_ll(sup, sh)};
    const int kinds2[4] = {0, 1, 1, 2};
    cluster_combine(red2, kinds2, 4, sh, cl, cs);
    const double gd = red2[0], stat = red2[1], hinf = red2[2];
    const long long support = (long long)red2[3];
    mark(7);

    if (a.mode != PROJ_ITER) {
      if (rank == 0 && threadIdx.x == 0) {
        st->theta = theta;
        st->support = support;
        st->h_inf = hinf;
        if (a.mode == PROJ_ALPHA0)
          st->alpha0 = hinf == 0.0 ? cfg.alpha_max : clamp_step(dvd(1.0, hinf), cfg);
      }
      break;
    }
    // escalation (gpss.cpp:169-191); every CTA takes the same decision
    if (attempt == 0) first_stat = stat;
    int outcome;  // 0 stationary, 1 accepted, 2 floor stop, 3 escalate
    if (stat <= st->stationarity_tol) outcome = 0;
    else if (gd < 0.0) outcome = 1;
    else if (alpha >= cfg.alpha_max) outcome = 2;
    else outcome = 3;
    if (outcome == 3) {
      const double a10 = mul(alpha, 10.0);
      alpha = a10 < cfg.alpha_max ? a10 : cfg.alpha_max;
      continue;
    }
    if (rank == 0 && threadIdx.x == 0) {
      st->out_stationarity = outcome == 2 ? first_stat : stat;
      if (outcome == 1) {
        st->alpha_used = alpha;
        st->stat = stat;
        st->gd = gd;
        st->theta = theta;
        st->support = support;
      } else {
        st->stationary = 1;
        st->status = STOPPED;
        st->reason = L1G_STATIONARY;
        l1g_iter_record& r = st->last;
        r.k = st->k;
        r.f = st->f;
        r.alpha = outcome == 2 ? first_alpha : alpha;
        r.stationarity = outcome == 2 ? first_stat : stat;
        r.step = nan_d();
        r.dir_derivative = outcome == 0 ? nan_d() : gd;
        r.theta = theta;
        r.support = support;
      }
    }
    break;
  }
  cl.sync();
}

// ---------------------------------------------------------------- host side
ProjPlan make_proj_plan(int64_t p_pad) {
  ProjPlan pp{};
  int cs = 1;
  while (cs < MAX_CS && (p_pad + cs - 1) / cs > 8192) cs <<= 1;
  int64_t per = (p_pad + cs - 1) / cs;
  int64_t ls = 32;
  while (ls < per) ls <<= 1;
  if (ls > MAX_LS) throw InvalidArgument("projection: p too large for the cluster kernel");
  pp.cs = cs;
  pp.ls = ls;
  const size_t budget = 227 * 1024 - sizeof(ProjShared) - 256;
  const int64_t cap = (int64_t)(budget / 8) - ls;
  int64_t c2 = 1;
  while (c2 * 2 <= cap) c2 <<= 1;
  pp.cand_cap = c2 < cap ? c2 + 1 : c2;
  if (pp.cand_cap > cap) pp.cand_cap = cap;
  pp.smem = (size_t)(ls + pp.cand_cap) * 8;
  return pp;
}

static int64_t pow2_at_least(int64_t v) {
  int64_t n = 1;
  while (n < v) n <<= 1;
  return n;
}

size_t proj_scratch_doubles(int64_t p_pad) {
  return (size_t)(pow2_at_least(p_pad) + 1) + (size_t)(p_pad + 2) + 64;
}

void launch_proj(const ProjPlan& pp, int mode, int64_t p, int64_t p_pad, const double* xin,
                 const double* gin, double* out, double* scratch, DevState* st,
                 const VecBufs* vb, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    L1G_CUDA(cudaFuncSetAttribute(proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(227 * 1024 - sizeof(ProjShared) - 64)));
    L1G_CUDA(cudaFuncSetAttribute(proj_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  ProjArgs a{};
  a.mode = mode;
  a.p = p;
  a.p_pad = p_pad;
  a.ls = pp.ls;
  a.cs = pp.cs;
  a.cand_cap = pp.cand_cap;
  a.xin = xin;
  a.gin = gin;
  a.out = mode == PROJ_ITER ? vb->d : out;
  a.gcand = scratch;
  a.gpre = scratch + pow2_at_least(p_pad) + 1;
  a.st = st;
  if (vb) a.vb = *vb;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pp.cs, 1, 1);
  cfg.blockDim = dim3(PT, 1, 1);
  cfg.dynamicSmemBytes = pp.smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = pp.cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  L1G_CUDA(cudaLaunchKernelEx(&cfg, proj_kernel, a));
}

}  // namespace l1g
