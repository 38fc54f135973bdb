// project.cu -- Euclidean projection onto the l1 ball as one thread-block cluster.
//
// Replaces project_l1_ball_with_threshold (prox.cpp:38-73) and, in PROJ_ITER mode, steps
// 1-3 of gp_iterate (gpss.cpp:146-192): steplength choice, v = x - alpha g, h = P(v),
// d = h - x, ||h - x||_inf, g'd and the alpha escalation loop, all on device.
//
// A cluster of `cs` CTAs (512 threads each) owns the vector; thread t of CTA r keeps the
// aligned run of M elements [r*ls + t*M, r*ls + (t+1)*M) in registers, so every canonical
// pairwise reduction is a register tree -> warp butterfly -> 16 warp values -> cs CTAs.
// The threshold is found without a host sort:
//   1. Michelot's pivot iteration (cluster-wide counts and sums) brackets theta from below;
//   2. the elements above the bracket plus the largest one below it are gathered into
//      CTA 0 and bitonic-sorted (shared memory, or L2-resident global memory if large);
//   3. one thread forms the *sequential* descending prefix sums exactly as prox.cpp:43-52
//      does, all threads test |v|_(k) > (S_k - rho)/k in parallel and the first failure
//      fixes theta -- bit-identical to the reference's sort-and-scan;
//   4. the feasibility bump loop of prox.cpp:58-65 on canonical cluster-wide l1 norms.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "engine.h"
#include "scalar.cuh"
#ifdef L1G_PROJ_TRACE  // debug builds only (tools/prof_solve.py --prefix-trace)
__device__ long long g_ptrace[192];
__device__ long long g_pstamp[65 * 8];
#define L1G_PREFIX_TRACE g_ptrace
#define L1G_PREFIX_STAMPS g_pstamp
#endif
#include "prefix.cuh"
#include "steps.cuh"

namespace cg = cooperative_groups;

namespace l1g {

#ifndef L1G_PROJ_KEEP  // keep x, g in registers between the first and the last pass up to this M
#define L1G_PROJ_KEEP 2
#endif
#ifndef L1G_PROJ_VS_MIN  // v lives in shared memory from this M up (see proj_kernel)
#define L1G_PROJ_VS_MIN 4
#endif
#ifndef L1G_PROJ_WARM
#define L1G_PROJ_WARM 0
#endif

constexpr int PT = 512;
constexpr int PW = PT / 32;
constexpr int MAX_M = 512;  // M > 32: v in global scratch (p up to 4 194 304)
constexpr int MAX_CS = 16;
constexpr int64_t SMEM_CAND = 16384;             // candidates sortable in shared memory

struct ProjArgs {
  int mode;
  int64_t p, p_pad, ls;
  int cs;
  int64_t cand_cap;
  const double* xin;
  const double* gin;
  double* out;
  double* gcand;  // global scratch: candidates (next_pow2(p_pad) + 1)
  double* gpre;   // global scratch: v of M > 32 plans (2 next_pow2(p_pad) + 2)
  DevState* st;
  VecBufs vb;
  // batched runs: cluster k projects problem k (vectors bstride apart, states consecutive)
  int64_t bstride, scr_stride;
  // sharded runs: per-rank packet scalars [nranks][SHARD_SCAL] (s'z, s's, z'z subtree values
  // of the rank's columns, its clock)
  const double* rank_scal;
  int nranks;
  // batched runs keep two plans in the iteration (one CTA per problem while many problems are
  // live, a cluster per problem once few are): this launch runs only if the live count *sel
  // is above (sel_mode 1) / at most (sel_mode 2) sel_thr
  const int* sel;
  int sel_thr, sel_mode;
};

struct ProjShared {
  double slot[2][MAX_CS][6];  // cluster exchange slots (double-buffered), filled by st.async
  uint64_t xbar[2];           // their mbarriers (complete_tx of every CTA's values)
  double wv[2][PW][6];         // warp partials (double-buffered)
  long long wl[PW][2];
  double bc[8];
  int dec;
};

// ---------------------------------------------------------------- distributed sort state
constexpr int NB = 256;  // key-bit bins of the cluster bucket sort (small M)
constexpr int NB_LARGE = 1024;  // M >= 16 (C4-class vectors: tens of thousands of candidates)
constexpr int RANK_MAXBIN = 256;  // largest bin the rank sort takes (else bitonic sorts)
constexpr int SMALL_RANK = 256;   // single-CTA path: rank sort up to this many candidates
#ifndef L1G_PREFIX_CLUSTER_MIN  // more candidates than this: the exact prefix runs cluster-wide
#define L1G_PREFIX_CLUSTER_MIN 8192
#endif
constexpr long long PREFIX_CLUSTER_MIN = L1G_PREFIX_CLUSTER_MIN;
#ifndef L1G_PREFIX_NT  // threads of the one-CTA exact prefix (fewer warps: cheaper barriers)
#define L1G_PREFIX_NT 512
#endif
constexpr int PREFIX_NT = L1G_PREFIX_NT;
template <int NBv>
struct SortShared {
  int hist[NBv];    // this CTA's candidates per bin
  int gcnt[NBv];    // cluster-wide candidates per bin
  int myoff[NBv];   // this CTA's offset inside each bin
  int start[NBv];   // global position of each bin (bins in descending value order)
  int cursor[NBv];
  int dest[NBv];
  int base[MAX_CS + 1];
  double next;
  int total, shift, ok, maxbin;
};

// ---------------------------------------------------------------- helpers
template <int M>
__device__ __forceinline__ int swz(int e) {  // bank-conflict-free thread-run layout
  constexpr int C = M >= 16 ? 15 : M - 1;
  const int t = e / M, k = e - t * M;
  return t * M + (k ^ (t & C));
}

// Parities of the double-buffered reduction buffers.  Every thread keeps its own copy (all
// threads run the same sequence of reductions), so no barrier is spent on flipping them, and
// a buffer is rewritten only after the barrier of the reduction in between.
struct RedPar {
  int b, c;     // block (warp partials), cluster (rank slots)
  unsigned ph;  // bit c: phase parity of the exchange mbarrier of slot buffer c
};

// Cluster exchange: every CTA sends nv doubles into slot[buf][its rank][0..nv) of every CTA
// with st.async, completing on that CTA's mbarrier xbar[buf]; a CTA proceeds once all cs * nv
// values have arrived.  One remote-store round trip instead of DSMEM stores + a full
// cluster barrier (954 vs 1669 cycles at cs = 16, tools/bench_cluster_sync.cu).  A buffer is
// rewritten two exchanges later, and any CTA's sends for exchange k + 2 follow its receipt of
// exchange k + 1, which every CTA sends only after reading exchange k: double-buffering is
// enough, provided every caller separates its reads of the slots from its next exchange by
// a block barrier (so no sender thread, tid < cs, runs ahead of a slow reader); all callers
// do.  Returns the buffer holding the values; every CTA must call it in the same order.
__device__ __forceinline__ int cluster_exchange(const double* vals, int nv, ProjShared& sh,
                                                cg::cluster_group& cl, int cs, RedPar& rp) {
  const unsigned rank = cl.block_rank();
  const int buf = rp.c;
  if (threadIdx.x == 0) mbar_arrive_expect_tx(&sh.xbar[buf], (uint32_t)(cs * nv * 8));
  if ((int)threadIdx.x < cs) {
    const uint32_t ra = mapa_u32(smem_u32(&sh.slot[buf][rank][0]), (int)threadIdx.x);
    const uint32_t rb = mapa_u32(smem_u32(&sh.xbar[buf]), (int)threadIdx.x);
    for (int c = 0; c < nv; ++c) st_async_f64(ra + 8u * c, vals[c], rb);
  }
  mbar_wait_cluster(&sh.xbar[buf], (rp.ph >> buf) & 1u);
  rp.ph ^= 1u << buf;
  rp.c ^= 1;
  return buf;
}

// Max over a warp of doubles that are >= 0 or exactly -1 (-1: none), as two 32-bit REDUX
// ops on the bit patterns (signed order of the high words, then the low words of the lanes
// holding the maximal high word) instead of five dependent shuffle + compare steps.
__device__ __forceinline__ double warp_max_nn(double v) {
  const long long b = __double_as_longlong(v);
  const int hi = (int)(b >> 32);
  const int mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)b : 0u);
  return __longlong_as_double((long long)(((unsigned long long)(unsigned)mhi << 32) | mlo));
}
// Sum over a warp of small non-negative integer counts held as doubles (REDUX)
__device__ __forceinline__ double warp_count(double v) {
  return (double)__reduce_add_sync(0xffffffffu, (unsigned)v);
}

// Several block reductions with one barrier.  kinds[c]: 0 = canonical tree over the threads'
// aligned runs (warp butterfly, then butterfly over the warp index), 1 = max (values >= 0 or
// -1), 2 = plain sum, 3 = count (integer-valued, < 2^32).
// Every thread receives the results.
template <int N>
__device__ __forceinline__ void block_reduce(double (&v)[N], const int (&kinds)[N],
                                             ProjShared& sh, RedPar& rp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const double x = kinds[c] == 1 ? warp_max_nn(v[c])
                                   : (kinds[c] == 3 ? warp_count(v[c]) : warp_tree(v[c]));
    if (lane == 0) sh.wv[rp.b][warp][c] = x;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double x = lane < PW ? sh.wv[rp.b][lane][c] : (kinds[c] == 1 ? -1.0 : 0.0);
    if (kinds[c] == 1) {
      v[c] = warp_max_nn(x);
    } else if (kinds[c] == 3) {
      v[c] = warp_count(x);
    } else {
#pragma unroll
      for (int o = 1; o < PW; o <<= 1) x = add(x, __shfl_xor_sync(0xffffffffu, x, o));
      v[c] = __shfl_sync(0xffffffffu, x, 0);
    }
  }
  rp.b ^= 1;
}

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
#pragma unroll
  for (int w = 0; w < PW; ++w) {
    const long long c = sh.wl[w][1];
    base += w < warp ? c : 0;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return base + inc - v;
}

// Cluster-wide combine of per-CTA values (identical in every thread of a CTA).  kinds[c]:
// 0 = canonical tree over ranks, 1 = max (>= 0 or -1), 2 = plain sum, 3 = count.  The values are exchanged into
// every CTA's slots (cluster_exchange), then every warp combines the local slots by a
// butterfly over the rank.  Every CTA must call it in the same order.
__device__ __forceinline__ void cluster_combine(double* vals, const int* kinds, int nv,
                                                ProjShared& sh, cg::cluster_group& cl, int cs,
                                                RedPar& rp) {
  if (cs == 1) return;
  const int buf = cluster_exchange(vals, nv, sh, cl, cs, rp);
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < nv; ++c) {
    double x = lane < cs ? sh.slot[buf][lane][c] : (kinds[c] == 1 ? -1.0 : 0.0);
    if (kinds[c] == 1) {
      vals[c] = warp_max_nn(x);
    } else if (kinds[c] == 3) {
      vals[c] = warp_count(x);
    } else {
      for (int o = 1; o < cs; o <<= 1) x = add(x, __shfl_xor_sync(0xffffffffu, x, o));
      vals[c] = __shfl_sync(0xffffffffu, x, 0);
    }
  }
}

// descending bitonic sort of n2 (power of two) values by the first min(PT, n2/2) threads
// (whole warps) of one CTA; the other threads return immediately.
template <class P>
__device__ void bitonic_desc(P c, int n2) {
  const int half = n2 >> 1;
  const int nthr = half >= PT ? PT : (half < 32 ? 32 : half);
  if ((int)threadIdx.x >= nthr) return;
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int pidx = threadIdx.x; pidx < half; pidx += nthr) {
        const int i = ((pidx & ~(j - 1)) << 1) | (pidx & (j - 1));
        const int ixj = i + j;
        const double a = c[i], b = c[ixj];
        const bool desc = (i & k) == 0;
        if (desc ? (a < b) : (a > b)) {
          c[i] = b;
          c[ixj] = a;
        }
      }
      if (nthr == 32) __syncwarp();
      else named_bar_sync(2, nthr);
    }
  }
}

// Pairwise tree over a thread's run of M leaves.  With v in shared memory (VS) the run is
// summed as 8-leaf subtrees pushed into a binary counter, so at most a few partial sums are
// live (a full unroll would hold all M leaves in registers); the value is the same tree.
template <int M, bool VS, class F>
__device__ __forceinline__ double run_tree(const F& leaf) {
  constexpr int L = M <= 128 ? 8 : (M <= 256 ? 9 : 10);  // the counter holds < 2^L leaves
  if constexpr (!VS || M <= 8) {
    return tree<M>(leaf);
  } else {
    Counter<L> c;
#pragma unroll 1
    for (int grp = 0; grp < M / 8; ++grp) c.template push_node<3>(tree<8>(leaf, grp * 8), (uint32_t)grp);
    return c.final_value((uint32_t)(M / 8) << 3);
  }
}

// LB coalesced elements j = tid + PT*(i0 + b) of x (and g when `wg`), every load issued before
// any is used: explicit global loads at a clamped (always valid) index, so the compiler keeps
// them in flight instead of interleaving them with the shared-memory staging stores.  Kept
// registers (KEEP) are used instead when the caller holds x and g already.
template <int LB, bool KEEP, int KM>
__device__ __forceinline__ void load_batch(double (&xb)[LB], double (&gb)[LB], const double (&xr)[KM],
                                           const double (&gr)[KM], const double* x, const double* g,
                                           int i0, int tid, int64_t base, int64_t lim, bool wg) {
#pragma unroll
  for (int b = 0; b < LB; ++b) {
    if (KEEP) {
      xb[b] = xr[KEEP ? i0 + b : 0];
      gb[b] = gr[KEEP ? i0 + b : 0];
    } else {
      const int64_t j = tid + (int64_t)PT * (i0 + b);
      const int64_t gj = j < lim ? base + j : 0;
      xb[b] = __ldcg(x + gj);
      gb[b] = wg ? __ldcg(g + gj) : 0.0;
    }
  }
}

// ---------------------------------------------------------------- cluster-wide exact prefix
// The sorted-prefix threshold search of prox.cpp:43-52 (see prefix_break in prefix.cuh for
// the arithmetic) over a candidate list distributed across the cluster: CTA r holds the
// descending run of global positions [B[r], E_r) in its own shared memory (E_r = B[r + 1],
// the last CTA's run extends to L), so the sorted candidates are never gathered into one
// CTA and every epoch's window is scanned by all CTAs that hold part of it.  Per epoch two
// cluster exchanges replace the block barriers of the one-CTA version: the CTAs' grid-count
// totals (or, with rounding ties, their parity segments) fix each CTA's exact running count,
// and the CTAs' first events (failure, binade exit, close call) give the window's first
// event.  Every CTA returns the same ff and S_{ff-1}.
__device__ __forceinline__ double cand_at(long long i, const int* B, int cs, double* cand,
                                          cg::cluster_group& cl) {
  int r = 0;
  while (r + 1 < cs && B[r + 1] <= i) ++r;
  return cl.map_shared_rank(cand, r)[i - B[r]];
}

__device__ long long prefix_break_cluster(double* cand, const int* B, int cs, long long L,
                                          double rho, ScanShared& ss, ProjShared& sh,
                                          cg::cluster_group& cl, RedPar& rp, double* s_before,
                                          double* pf) {
  long long t_pf = clock64();
  auto pmark = [&](int idx) {  // sub-phase cycles into pf[idx] (CTA 0, thread 0 only)
    if (pf) {
      const long long t = clock64();
      pf[idx] += (double)(t - t_pf);
      t_pf = t;
    }
  };
  constexpr int NW = PT / 32;
  constexpr long long TWO53 = 1LL << 53;
  constexpr unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  if (L <= 0) {
    *s_before = 0.0;
    return 0;
  }
  // ---- head (CTA 0): the reference's own sequential adds over the first H positions
  const int H = L < PREFIX_HEAD ? (int)L : PREFIX_HEAD;
  {
    double hv[3] = {-1.0, 0.0, 0.0};  // first failure (or -1), S_{H-1}, S before the failure
    if (rank == 0) {
      const double m = tid < H ? cand_at(tid, B, cs, cand, cl) : 0.0;
      if (tid < PREFIX_HEAD) ss.head[tid] = m;
      __syncthreads();
      if (tid == 0) head_sums(ss.head, H);
      __syncthreads();
      const bool bad = tid < H && !passes(m, ss.head[tid], rho, tid + 1);
      const unsigned bb = __ballot_sync(FULL, bad);
      if (lane == 0) ss.hbad[warp] = bb ? warp * 32 + __ffs(bb) - 1 : INT_MAX;
      __syncthreads();
      int ff = INT_MAX;
#pragma unroll
      for (int w = 0; w < NW; ++w) ff = min(ff, ss.hbad[w]);
      hv[0] = ff == INT_MAX ? -1.0 : (double)ff;
      hv[1] = ss.head[H - 1];
      hv[2] = ff == INT_MAX ? 0.0 : (ff > 0 ? ss.head[ff - 1] : 0.0);
    }
    pmark(24);
    const int xb = cluster_exchange(hv, 3, sh, cl, cs, rp);
    const double hf = sh.slot[xb][0][0];
    pmark(27);
    if (hf >= 0.0 || H == L) {
      if (tid == 0) ss.epochs = 0;
      *s_before = hf >= 0.0 ? sh.slot[xb][0][2] : sh.slot[xb][0][1];
      return hf >= 0.0 ? (long long)hf : L;
    }
    hv[1] = sh.slot[xb][0][1];
    __syncthreads();  // every thread read the slots before the next exchange
    double S_prev = hv[1];
    // ---- epochs
    const long long Br = B[rank], Er = rank == cs - 1 ? L : B[rank + 1];
    const double* c = cand - Br;  // c[i] for global positions i in [Br, Er)
    long long i0 = H, window = 2 * H;
    int par = 0, nep = 0;
    while (i0 < L) {
      ++nep;
      if (!(S_prev >= 0x1.0p-960)) {  // (sub)tiny running sum: one scalar step, uniform
        const double ci = cand_at(i0, B, cs, cand, cl);
        const double S = add(S_prev, ci);
        if (!passes(ci, S, rho, i0 + 1)) {
          *s_before = S_prev;
          if (tid == 0) ss.epochs = nep;
          return i0;
        }
        S_prev = S;
        ++i0;
        continue;
      }
      const long long n = (L - i0) < window ? (L - i0) : window;
      const long long wend = i0 + n;
      const long long lo = i0 > Br ? i0 : Br, hi = wend < Er ? wend : Er;
      const long long len = hi > lo ? hi - lo : 0;
      const long long E = (len + PT - 1) / PT;
      const long long p0 = lo + tid * E < hi ? lo + tid * E : hi;
      const long long p1 = p0 + E < hi ? p0 + E : hi;
      const long long sbits = __double_as_longlong(S_prev);
      const int be = (int)(sbits >> 52);
      const long long base_q = (sbits & ((1LL << 52) - 1)) | (1LL << 52);
      // pass 1: this thread's grid counts; CTA totals (or parity segments with ties)
      long long qs = 0;
      bool anytie = false;
      for (long long i = p0; i < p1; ++i) {
        bool t;
        qs += grid_count(c[i], be, &t);
        anytie |= t;
      }
      const unsigned tball = __ballot_sync(FULL, anytie);
      long long qinc = qs;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(FULL, qinc, o);
        if (lane >= o) qinc += y;
      }
      if (lane == 31) {
        ss.fq[par][warp] = qinc;
        ss.ftie[par][warp] = tball != 0;
      }
      __syncthreads();
      pmark(25);
      long long wex = 0, tot = 0;
      int ties = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const long long d = ss.fq[par][w];
        wex += w < warp ? d : 0;
        tot += d;
        ties |= ss.ftie[par][w];
      }
      ParSeg cta = seg_elem(tot, false), incl = seg_id();  // the CTA's run; this thread's (ties)
      if (ties) {  // uniform over the CTA
        ParSeg me = seg_id();
        for (long long i = p0; i < p1; ++i) {
          bool t;
          const long long q = grid_count(c[i], be, &t);
          me = seg_then(me, seg_elem(q, t));
        }
        incl = seg_warp_scan(me, lane);
        if (lane == 31) {
          ss.wd0[par][warp] = incl.d0;
          ss.wpk[par][warp] = seg_pack(incl);
        }
        __syncthreads();
        cta = seg_id();
#pragma unroll
        for (int w = 0; w < NW; ++w) cta = seg_then(cta, seg_unpack(ss.wd0[par][w], ss.wpk[par][w]));
      }
      pmark(26);
      // exchange 1: the CTAs' segments -> this CTA's exact starting count and the window's end
      double xs[2] = {__longlong_as_double(cta.d0), (double)seg_pack(cta)};
      const int x1 = cluster_exchange(xs, 2, sh, cl, cs, rp);
      pmark(27);
      long long Nr = base_q, Nend = base_q;
      for (int r = 0; r < cs; ++r) {
        const ParSeg sr = seg_unpack(__double_as_longlong(sh.slot[x1][r][0]), (int)sh.slot[x1][r][1]);
        Nr = r == rank ? Nend : Nr;
        Nend = seg_apply(sr, Nend);
      }
      long long N;
      if (ties) {  // the warps' starts, then the lanes' within the warp
        long long Nw = Nr;
        long long acc = Nr;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const ParSeg sw = seg_unpack(ss.wd0[par][w], ss.wpk[par][w]);
          Nw = w == warp ? acc : Nw;
          acc = seg_apply(sw, acc);
        }
        ParSeg ex = seg_shfl_up(incl, 1);
        if (lane == 0) ex = seg_id();
        N = seg_apply(ex, Nw);
      } else {
        N = Nr + wex + (qinc - qs);
      }
      // pass 2: exact sums and tests; this thread's first event
      int my_ev = INT_MAX, kind = 0;
      long long my_n = 0;
      double kd = (double)(p0 + 1);
      for (long long i = p0; i < p1; ++i) {
        const double m = c[i];
        bool tie;
        const long long q = grid_count(m, be, &tie);
        const long long Nn = N + q + (tie ? ((N + q) & 1) : 0);
        const int stt = Nn >= TWO53 ? 2 : quick_test(m, from_grid(Nn, be), rho, kd);
        const bool take = stt != 0 && my_ev == INT_MAX;
        my_ev = take ? (int)i : my_ev;
        kind = take ? stt : kind;
        my_n = take ? N : my_n;
        N = Nn;
        kd = add(kd, 1.0);
      }
      const unsigned have = __ballot_sync(FULL, my_ev != INT_MAX);
      if (have) {
        if (lane == __ffs(have) - 1) {
          ss.epos[par][warp] = my_ev;
          ss.ekind[par][warp] = kind;
          ss.en[par][warp] = my_n;
        }
      } else if (lane == 0) {
        ss.epos[par][warp] = INT_MAX;
      }
      __syncthreads();
      int ew = -1;
#pragma unroll
      for (int w = NW - 1; w >= 0; --w) ew = ss.epos[par][w] != INT_MAX ? w : ew;
      pmark(28);
      // exchange 2: the CTAs' first events -> the window's first event
      double xe[4] = {-1.0, 0.0, 0.0, 0.0};
      if (ew >= 0) {
        const int ev = ss.epos[par][ew];
        xe[0] = (double)ev;
        xe[1] = (double)ss.ekind[par][ew];
        xe[2] = __longlong_as_double(ss.en[par][ew]);
        xe[3] = c[ev];
      }
      const int x2 = cluster_exchange(xe, 4, sh, cl, cs, rp);
      pmark(29);
      int er = -1;
      for (int r = cs - 1; r >= 0; --r) er = sh.slot[x2][r][0] >= 0.0 ? r : er;  // lowest rank
      par ^= 1;
      if (er < 0) {  // the whole window is exact and passes: the epoch continues
        S_prev = from_grid(Nend, be);
        i0 = wend;
        window *= 2;
        __syncthreads();  // slots read before the next exchange
        continue;
      }
      const long long ev = (long long)sh.slot[x2][er][0];
      const int evk = (int)sh.slot[x2][er][1];
      const long long nb = __double_as_longlong(sh.slot[x2][er][2]);
      const double cev = sh.slot[x2][er][3];
      __syncthreads();  // slots read before the next exchange
      const double sb = from_grid(nb, be);  // S_{ev-1}
      if (evk == 1) {
        *s_before = sb;
        if (tid == 0) ss.epochs = nep;
        return ev;
      }
      if (evk == 3) {  // exact test with the division; on success the epoch goes on
        bool t;
        const long long qe = grid_count(cev, be, &t);
        const double Se = from_grid(nb + qe + (t ? ((nb + qe) & 1) : 0), be);
        if (!passes(cev, Se, rho, ev + 1)) {
          *s_before = sb;
          if (tid == 0) ss.epochs = nep;
          return ev;
        }
        S_prev = Se;
        i0 = ev + 1;
        continue;
      }
      const double S = add(sb, cev);  // the binade exit: one IEEE addition
      if (!passes(cev, S, rho, ev + 1)) {
        *s_before = sb;
        if (tid == 0) ss.epochs = nep;
        return ev;
      }
      window = ((2 * (ev + 1) + 31) >> 5) << 5;
      S_prev = S;
      i0 = ev + 1;
    }
    *s_before = S_prev;
    if (tid == 0) ss.epochs = nep;
    return L;
  }
}

__device__ __forceinline__ double soft(double v, double th) {
  return v > th ? sub(v, th) : (v < -th ? add(v, th) : 0.0);
}

// ---------------------------------------------------------------- the kernel
#ifdef L1G_TIMELINE
__device__ unsigned long long g_tl_proj[256 * 16];
#endif

template <int M>
__global__ void __launch_bounds__(PT, 1) proj_kernel(const ProjArgs a) {
  L1G_TL_ENTRY
  pdl_wait_and_trigger();
  L1G_TL_WAITED(a.mode == PROJ_ITER && blockIdx.x == 0, g_tl_proj, 0, a.st->k)
  if (a.sel_mode != 0) {  // the other plan's launch takes this iteration (uniform over the grid)
    const int live = __ldcg(a.sel);
    if ((a.sel_mode == 1) != (live > a.sel_thr)) return;
  }
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int cs = a.cs;
  constexpr int64_t LS = (int64_t)PT * M;
  extern __shared__ __align__(16) double dyn[];  // staging (LS) / CTA 0 candidates
  __shared__ ProjShared sh;
  __shared__ ScanShared scan_sh;
  __shared__ DevState sst;
  // key-bit bins: enough that the bins stay narrow for the rank sort on large vectors
  constexpr int NBK = M >= 16 ? NB_LARGE : NB;
  __shared__ SortShared<NBK> srt;
  const int prob = (int)(blockIdx.x / (unsigned)a.cs);
  const int64_t pofs = prob * a.bstride;
  DevState* st = a.st + prob;
  const int tid = threadIdx.x;
  RedPar rp{0, 0, 0u};
  const bool prof = (a.mode == PROJ_ITER) && rank == 0 && tid == 0;
  long long t_last = clock64();
  auto mark = [&](int idx) {
    if (prof) {
      const long long t = clock64();
      sst.prof[idx] += (double)(t - t_last);
      t_last = t;
    }
  };
  auto count = [&](int idx, double v) {
    if (prof) sst.prof[idx] += v;
  };
  // one coalesced copy of the device state instead of many dependent scalar loads
  {
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sst);
    for (int i = tid; i < (int)(sizeof(DevState) / 8); i += PT) dst[i] = src[i];
  }
  if (tid == 0) {
    mbar_init(&sh.xbar[0], 1);
    mbar_init(&sh.xbar[1], 1);
    fence_barrier_init();  // visible cluster-wide before the first cluster barrier
  }
  __syncthreads();
  if (a.mode == PROJ_ITER && sst.status != RUNNING) return;  // uniform over the cluster
  // every CTA of the cluster is running before any DSMEM access (PROJ_ITER: the barrier of
  // the steplength broadcast below)
  if (a.mode != PROJ_ITER && cs > 1) cl.sync();
  const l1g_gp_config cfg = sst.cfg;
  const double rho = sst.rho;
  const int cur = a.mode == PROJ_ITER ? sst.cur : 0;
  const double* x = (a.mode == PROJ_ITER ? a.vb.x[cur] : a.xin) + pofs;
  const double* g = (a.mode == PROJ_ITER ? a.vb.g[cur] : a.gin) + pofs;
  double* const dout = a.out + pofs;
  double* const gcand = a.gcand + prob * a.scr_stride;
  const int64_t base = (int64_t)rank * LS;
  const int64_t lim = a.p_pad - base < LS ? (a.p_pad - base > 0 ? a.p_pad - base : 0) : LS;

  // ---- steplength and loop-top checks (gpss.cpp:233-245, :147-153), CTA 0 decides
  double alpha = 1.0, first_alpha = 1.0;
  if (a.mode == PROJ_ITER) {
    if (rank == 0 && tid == 0) {
      int dec = 0;
      double el = 0.0;
      if (a.nranks > 1) {
        // column shards: the secant dots are the canonical tree over the ranks' subtree
        // values (shard widths are equal powers of two, so the ranks' subtrees are the
        // canonical column tree's), and every rank takes the budget decision on the same
        // clock -- the latest any rank reported -- so all ranks stop on the same iteration
        double t3[3][16];
        for (int r = 0; r < a.nranks; ++r) {
          for (int c = 0; c < 3; ++c) t3[c][r] = a.rank_scal[r * SHARD_SCAL + c];
          el = fmax(el, a.rank_scal[r * SHARD_SCAL + 3]);
        }
        for (int h = 1; h < a.nranks; h <<= 1)
          for (int i = 0; i + h < a.nranks; i += 2 * h)
            for (int c = 0; c < 3; ++c) t3[c][i] = add(t3[c][i], t3[c][i + h]);
        sst.sz = t3[0][0];
        sst.ss = t3[1][0];
        sst.zz = t3[2][0];
        st->sz = sst.sz;
        st->ss = sst.ss;
        st->zz = sst.zz;
      } else {
        el = sst.max_seconds > 0.0 ? elapsed_s(&sst) : 0.0;
      }
      if (!sst.single_step) {
        if (sst.max_iterations > 0 && sst.k >= sst.max_iterations) dec = 1 + L1G_MAX_ITERATIONS;
        else if (sst.max_matvecs > 0 && sst.matvecs >= sst.max_matvecs) dec = 1 + L1G_MAX_MATVECS;
        else if (sst.max_seconds > 0.0 && el >= sst.max_seconds) dec = 1 + L1G_MAX_SECONDS;
      } else if (sst.stationary) {
        dec = 1 + L1G_STATIONARY;
      }
      double al = sst.alpha0;
      if (dec == 0) {
        l1g_sl_choice c;
        if (sst.k == 0) {
          c.alpha = sst.alpha0;
          c.bb_active = 0;
          c.bb1_raw = c.bb2_raw = c.tau_before = c.tau_after = nan_d();
        } else {
          steplength_from_dots(&sst.tau, sst.a2h, &sst.a2_len, sst.sz, sst.ss, sst.zz, cfg, &c);
          st->tau = sst.tau;
          for (int i = 0; i < sst.a2_len; ++i) st->a2h[i] = sst.a2h[i];
          st->a2_len = sst.a2_len;
        }
        st->choice = c;
        al = c.alpha;
      } else {
        st->reason = dec - 1;
        leave_run(st, STOPPED);
        if (dec - 1 == L1G_STATIONARY) {
          st->last.stationarity = 0.0;
          st->out_stationarity = 0.0;
        }
      }
      sh.bc[6] = al;
      sh.dec = dec;
    }
    cl.sync();
    if (tid == 0 && rank != 0) {
      const ProjShared* r0 = cl.map_shared_rank(&sh, 0);
      sh.bc[6] = r0->bc[6];
      sh.dec = r0->dec;
    }
    __syncthreads();  // (CTA 0 rewrites bc / dec only after later cluster barriers)
    if (sh.dec != 0) {
      cl.sync();  // no CTA leaves while another may still read its shared memory
      return;
    }
    alpha = first_alpha = sh.bc[6];
  }

  double first_stat = 0.0;
  count(8, 1.0);
  mark(0);
  // v = x - alpha g: in registers (thread-run order) for small M; in shared memory for
  // M >= 16, where 2M registers for v would leave too few for the rest and spill
  constexpr bool VS = M >= L1G_PROJ_VS_MIN;
  constexpr int UK = VS ? 4 : M;  // unroll of the passes over v (register arrays need all M)
  double vr[VS ? 1 : M] = {};
  // beyond M = 32 (p > 262 144) v does not fit in shared memory beside the candidates: it
  // lives in the L2-resident global scratch, the CTA's slice at its cluster offset
  constexpr bool VGLOB = M > 32;
  double* const vbuf = VGLOB ? a.gpre + prob * a.scr_stride + base : dyn;
  double* const cand = dyn + ((VS && !VGLOB) ? LS : 0);  // candidate buffer (sort, gather, prefix)
  auto VG = [&](int k) -> double { return VS ? vbuf[swz<M>(tid * M + k)] : vr[VS ? 0 : k]; };
  auto VSET = [&](int k, double val) {
    if (VS) vbuf[swz<M>(tid * M + k)] = val;
    else vr[VS ? 0 : k] = val;
  };
  // x and g in the coalesced order (j = tid + PT*i), kept for the final pass when small
  constexpr bool KEEP = M <= L1G_PROJ_KEEP;
  constexpr int LB = M < 8 ? M : 8;  // loads in flight per vector and thread
  constexpr int UB = VS ? 1 : M / LB;  // batches unrolled (VS: one batch's addresses live)
  constexpr int UBV = VS ? (M >= 32 ? 2 : 1) : M / LB;  // the first pass: two for M = 32
  double xr[KEEP ? M : 1], gr[KEEP ? M : 1];
  if (KEEP) {
#pragma unroll
    for (int i = 0; i < (KEEP ? M : 1); ++i) {
      const int64_t j = tid + (int64_t)PT * i;
      const bool in = j < lim;
      xr[i] = in ? x[base + j] : 0.0;
      gr[i] = in && a.mode != PROJ_PLAIN ? g[base + j] : 0.0;
    }
  }
  for (int attempt = 0;; ++attempt) {
    count(9, 1.0);
    // ---- v = x - alpha g  (gpss.cpp:167; alpha0: x0 - grad, gpss.cpp:95): coalesced
    //      loads (issued in batches of LB per vector, all in flight before the first use),
    //      staged through shared memory into per-thread registers
#pragma unroll UBV
    for (int i0 = 0; i0 < M; i0 += LB) {
      double xb[LB], gb[LB];
      load_batch<LB, KEEP>(xb, gb, xr, gr, x, g, i0, tid, base, lim, a.mode != PROJ_PLAIN);
#pragma unroll
      for (int b = 0; b < LB; ++b) {
        const int64_t j = tid + (int64_t)PT * (i0 + b);
        double val = 0.0;
        if (j < lim) {
          if (a.mode == PROJ_PLAIN) val = xb[b];
          else if (a.mode == PROJ_ALPHA0) val = sub(xb[b], gb[b]);
          else val = sub(xb[b], mul(alpha, gb[b]));
        }
        vbuf[swz<M>((int)j)] = val;
      }
    }
    __syncthreads();
    if (!VS) {
#pragma unroll
      for (int k = 0; k < M; ++k) VSET(k, vbuf[swz<M>(tid * M + k)]);
    }
    __syncthreads();
    double red[2];
    {
      const double t = run_tree<M, VS>([&](int k) { return fabs(VG(k)); });
      double m = 0.0;
#pragma unroll UK
      for (int k = 0; k < M; ++k) m = fmax(m, fabs(VG(k)));
      red[0] = t;
      red[1] = m;
      const int kinds[2] = {0, 1};
      block_reduce<2>(red, kinds, sh, rp);
      cluster_combine(red, kinds, 2, sh, cl, cs, rp);
    }
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
      // Michelot pivot iteration from below: th_{t+1} = (sum_{|v|>th_t} |v| - rho) / count
      // Warm start from the previous iteration's theta: each update is a Newton step on
      // the convex f(t) = sum max(|v|-t, 0) - rho, so a start above theta* lands at or below
      // it in one step and the iteration then climbs monotonically.  Only the bracket
      // depends on this; the exact sort-and-scan below decides theta.
      const double th_cold = dvd(sub(l1v, rho), (double)a.p_pad);
      bool warm = L1G_PROJ_WARM && a.mode == PROJ_ITER && sst.k > 0 && sst.theta > th_cold &&
                  sst.theta < vinf;
      double th = warm ? sst.theta : th_cold;
      double cnt_prev = (double)a.p_pad + 1.0;
      const int kinds_cs[2] = {3, 2};
      for (int it = 0; it < 64; ++it) {
        double v2[2] = {0.0, 0.0};
#pragma unroll UK
        for (int k = 0; k < M; ++k) {
          const double m = fabs(VG(k));
          if (m > th) {
            v2[0] += 1.0;
            v2[1] += m;
          }
        }
        block_reduce<2>(v2, kinds_cs, sh, rp);
        cluster_combine(v2, kinds_cs, 2, sh, cl, cs, rp);
        count(10, 1.0);
        if (warm) {  // first step from the previous theta
          warm = false;
          if (v2[0] == 0.0) {
            th = th_cold;
            continue;
          }
          const double thn = dvd(sub(v2[1], rho), v2[0]);
          if (thn < th) {  // started above theta*: restart the monotone climb from thn
            th = thn;
            continue;
          }
        }
        if (v2[0] == 0.0 || v2[0] >= cnt_prev) break;
        const double shrink = cnt_prev - v2[0];
        cnt_prev = v2[0];
        th = dvd(sub(v2[1], rho), v2[0]);
        if (shrink * 64.0 <= v2[0]) break;  // converged to within ~1.5% of the support
      }
      mark(2);
      // exact sort-and-scan on the elements above a bracket below theta
      double lo = th > 0.0 ? sub(th, mul(th, 0x1.0p-20)) : -1.0;
      for (int tries = 0;; ++tries) {
        long long myc = 0;
        double mynext = -1.0;
#pragma unroll UK
        for (int k = 0; k < M; ++k) {
          const double m = fabs(VG(k));
          if (m > lo) ++myc;
          else mynext = fmax(mynext, m);
        }
        long long ctot;
        const long long off = block_excl_scan(myc, sh, &ctot);
        double bnx[1] = {mynext};
        const int k_max[1] = {1};
        block_reduce<1>(bnx, k_max, sh, rp);
        const double bnext = bnx[0];
        long long before = 0, total = ctot;
        double next = bnext;
        if (cs > 1) {  // counts and the next value below the bracket, pushed to every CTA
          const double xv[2] = {(double)ctot, bnext};  // counts < 2^53: exact
          const int xb = cluster_exchange(xv, 2, sh, cl, cs, rp);
          long long b = 0, tt = 0;
          double nx = -1.0;
          for (int r = 0; r < cs; ++r) {
            const long long cr = (long long)sh.slot[xb][r][0];
            b += r < (int)rank ? cr : 0;
            tt += cr;
            nx = fmax(nx, sh.slot[xb][r][1]);
          }
          before = b;
          total = tt;
          next = nx;
        }
        const long long L = total + (next >= 0.0 ? 1 : 0);
        mark(14);
        if (cs > 1 && lo >= 0.0) {
          // ---- cluster bucket sort: bins on the key bits (~log scale), whole bins to CTAs,
          //      DSMEM scatter, local bitonic sorts, then the sorted ranges are gathered into
          //      CTA 0's shared memory (or, beyond its capacity, into the global scratch)
          const long long kmin = __double_as_longlong(lo);
          const long long kspan = __double_as_longlong(vinf) - kmin;  // candidates: key > kmin
          if (tid == 0) {
            int sh_ = 0;
            while ((kspan >> sh_) >= NBK) ++sh_;
            srt.shift = sh_;
          }
          for (int t = tid; t < NBK; t += PT) {
            srt.hist[t] = 0;
            srt.cursor[t] = 0;
          }
          __syncthreads();
          const int shft = srt.shift;
#pragma unroll UK
          for (int k = 0; k < M; ++k) {
            const double m = fabs(VG(k));
            if (m > lo) atomicAdd(&srt.hist[(int)((__double_as_longlong(m) - kmin) >> shft)], 1);
          }
          cl.sync();
          mark(21);
          for (int t = tid; t < NBK; t += PT) {
            int h[MAX_CS];
#pragma unroll
            for (int r = 0; r < MAX_CS; ++r)
              h[r] = r < cs ? cl.map_shared_rank(&srt, r)->hist[t] : 0;
            int gsum = 0, mine = 0;
#pragma unroll
            for (int r = 0; r < MAX_CS; ++r) {
              gsum += h[r];
              mine += r < (int)rank ? h[r] : 0;
            }
            srt.gcnt[t] = gsum;
            srt.myoff[t] = mine;
          }
          __syncthreads();
          mark(22);
          if (tid < 32) {  // descending exclusive scan over bins, destination CTAs
            const int lane = tid;
            int carry = 0, mx = 0;
            for (int c0 = NBK - 32; c0 >= 0; c0 -= 32) {
              const int b = c0 + 31 - lane;  // lane 0 takes the highest bin of the chunk
              int x = srt.gcnt[b], inc = x;
              mx = max(mx, x);
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
              }
              srt.start[b] = carry + inc - x;
              carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            const int share = (carry + cs - 1) / cs;
            for (int b = lane; b < NBK; b += 32) {
              const int d = share > 0 ? srt.start[b] / share : 0;
              srt.dest[b] = d < cs ? d : cs - 1;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) {
              srt.total = carry;
              srt.maxbin = mx;
            }
          }
          __syncthreads();
          {  // base[d] = first position owned by CTA d: one warp per d, min over bins
            const int w = tid >> 5, lane = tid & 31;
            if (w < cs) {
              int bmin = srt.total;
              for (int b = lane; b < NBK; b += 32)
                if (srt.dest[b] >= w && srt.gcnt[b] > 0) bmin = min(bmin, srt.start[b]);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
              if (lane == 0) srt.base[w] = w == 0 ? 0 : bmin;
            }
            if (tid == 0) srt.base[cs] = srt.total;
          }
          __syncthreads();
          if (tid == 0) {
            int ok = 1;
            for (int d = 0; d < cs; ++d) {
              if (srt.base[d + 1] < srt.base[d]) srt.base[d + 1] = srt.base[d];
              if (srt.base[d + 1] - srt.base[d] + 1 > a.cand_cap) ok = 0;
            }
            srt.ok = ok;
          }
          __syncthreads();
          mark(15);
          if (srt.ok) {
#pragma unroll UK
            for (int k = 0; k < M; ++k) {
              const double m = fabs(VG(k));
              if (m > lo) {
                const int b = (int)((__double_as_longlong(m) - kmin) >> shft);
                const int d = srt.dest[b];
                const int pos = srt.start[b] + srt.myoff[b] + atomicAdd(&srt.cursor[b], 1) - srt.base[d];
                cl.map_shared_rank(cand, d)[pos] = m;
              }
            }
          }
          cl.sync();
          mark(16);
          if (srt.ok) {
            // each CTA sorts its own range of global positions [base[r], base[r + 1]) in place;
            // the exact prefix then runs over the distributed ranges (prefix_break_cluster)
            const int cnt = srt.base[rank + 1] - srt.base[rank];
            constexpr int RK = M >= 16 ? 8 : 2;  // candidates per thread on the rank path
            int maxcnt = 0;  // the path must be the same in every CTA (cluster barriers)
            for (int d = 0; d < cs; ++d) maxcnt = max(maxcnt, srt.base[d + 1] - srt.base[d]);
            if (maxcnt <= RK * PT && srt.maxbin <= RANK_MAXBIN) {
              // rank sort: bins are narrow, so an element's place is its bin's start plus the
              // number of larger bin mates (equal ones ordered by position)
              const int b0 = srt.base[rank];
              double mv[RK];
              int pos[RK];
#pragma unroll
              for (int k = 0; k < RK; ++k) {
                const int i = tid + k * PT;
                pos[k] = -1;
                mv[k] = 0.0;
                if (i < cnt) {
                  const double m = cand[i];
                  const int b = (int)((__double_as_longlong(m) - kmin) >> shft);
                  const int s0 = srt.start[b] - b0, s1 = s0 + srt.gcnt[b];
                  int r = 0;
                  for (int j = s0; j < s1; ++j) {
                    const double y = cand[j];
                    r += (y > m) | ((y == m) & (j < i));
                  }
                  mv[k] = m;
                  pos[k] = srt.start[b] + r - b0;
                }
              }
              __syncthreads();  // the range is rewritten in place
              mark(17);
#pragma unroll
              for (int k = 0; k < RK; ++k)
                if (pos[k] >= 0) cand[pos[k]] = mv[k];
            } else {
              int m2 = 1;
              while (m2 < cnt) m2 <<= 1;
              for (int i = cnt + tid; i < m2; i += PT) cand[i] = 0.0;
              __syncthreads();
              if (cnt > 1) bitonic_desc(cand, m2);
              mark(17);
            }
            __syncthreads();
            long long ff;
            double s_before = 0.0;
            count(11, (double)total);
            if (total > PREFIX_CLUSTER_MIN) {
              // the largest element below the bracket closes the list (position `total`)
              if (rank == (unsigned)(cs - 1) && tid == 0 && next >= 0.0) cand[cnt] = next;
              cl.sync();  // every range final before other CTAs read it
              mark(3);
              ff = prefix_break_cluster(cand, srt.base, cs, L, rho, scan_sh, sh, cl, rp,
                                        &s_before, prof ? sst.prof : nullptr);
            } else {
              // few candidates: the per-epoch cluster exchanges would cost more than they
              // save; the ranges are gathered into CTA 0, which scans them alone
              cl.sync();  // every range sorted
              if (rank != 0) {
                double* dst = cl.map_shared_rank(cand, 0) + srt.base[rank];
                for (int i = tid; i < cnt; i += PT) dst[i] = cand[i];
              }
              if (rank == (unsigned)(cs - 1) && tid == 0 && next >= 0.0)
                cl.map_shared_rank(cand, 0)[total] = next;
              cl.sync();
              mark(3);
              double res[2] = {0.0, 0.0};
              if (rank == 0 && tid < PREFIX_NT)  // (the senders, tid < cs, are among them)
                res[0] = (double)prefix_break<PREFIX_NT>(cand, L, rho, scan_sh, &res[1]);
              const int xb = cluster_exchange(res, 2, sh, cl, cs, rp);
              ff = (long long)sh.slot[xb][0][0];
              s_before = sh.slot[xb][0][1];
            }
            count(20, (double)scan_sh.epochs);
            mark(5);
            // theta = candidate of the last passing index (prox.cpp:47-50); 0 if none passed.
            // All passed although smaller elements exist: the bracket was too high.
            if (!(ff == L && next >= 0.0)) {
              theta = ff > 0 ? dvd(sub(s_before, rho), (double)ff) : 0.0;
              break;
            }
            count(13, 1.0);
            lo = (lo > 0.0 && tries < 4) ? mul(lo, 0.5) : -1.0;
            continue;
          }
          // bins too unbalanced for the shared-memory ranges: single-CTA path below
        }
        int64_t n2 = 1;
        while (n2 < total) n2 <<= 1;
        const bool in_smem = (n2 + 1 <= a.cand_cap);
        double* cbuf = in_smem ? cl.map_shared_rank(cand, 0) : gcand;
        long long pos = before + off;
#pragma unroll UK
        for (int k = 0; k < M; ++k) {
          const double m = fabs(VG(k));
          if (m > lo) cbuf[pos++] = m;
        }
        if (!in_smem) __threadfence();
        cl.sync();
        mark(3);
        count(11, (double)total);
        if (rank == 0) {
          double* c = in_smem ? cand : gcand;
          if (total <= SMALL_RANK) {
            // few candidates: each one's place is the number of larger ones (equal ones by
            // position), one thread per candidate, every read a shared-memory broadcast
            double m = 0.0;
            int r = 0;
            if (tid < total) {
              m = c[tid];
              for (int j = 0; j < (int)total; ++j) {
                const double y = c[j];
                r += (y > m) | ((y == m) & (j < tid));
              }
            }
            __syncthreads();
            if (tid < total) c[r] = m;
          } else {
            for (int64_t i = total + tid; i < n2; i += PT) c[i] = 0.0;
            __syncthreads();
            bitonic_desc(c, (int)n2);
          }
          __syncthreads();
          if (tid == 0 && next >= 0.0) c[total] = next;
          __syncthreads();
          mark(4);
          double s_before = 0.0;
          const long long ff =
              tid < PREFIX_NT ? prefix_break<PREFIX_NT>(c, L, rho, scan_sh, &s_before) : 0;
          count(20, (double)scan_sh.epochs);
          if (tid == 0) {
            // theta = candidate of the last passing index (prox.cpp:47-50); 0 if none passed
            sh.bc[4] = ff > 0 ? dvd(sub(s_before, rho), (double)ff) : 0.0;
            // all passed although smaller elements exist: the bracket was too high
            sh.dec = (ff == L && next >= 0.0) ? 1 : 0;
          }
          mark(5);
          __syncthreads();
          if (tid > 0 && tid < cs) {  // push theta and the decision to the other CTAs
            ProjShared* dst = cl.map_shared_rank(&sh, tid);
            dst->bc[4] = sh.bc[4];
            dst->dec = sh.dec;
          }
        }
        if (cs > 1) cl.sync();
        else __syncthreads();
        if (!sh.dec) {
          theta = sh.bc[4];
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
        const double thc = theta;
        double l1u[1] = {run_tree<M, VS>([&](int k) { return fabs(soft(VG(k), thc)); })};
        block_reduce<1>(l1u, k_sum, sh, rp);
        cluster_combine(l1u, k_sum, 1, sh, cl, cs, rp);
        if (!(l1u[0] > rho && guard++ < 64)) break;
        count(12, 1.0);
        theta = add(theta, bump);
        bump = mul(bump, 2.0);
      }
      mark(6);
    }

    // ---- h, d = h - x, ||h - x||_inf, g'd, support  (gpss.cpp:167-178)
    const double th = theta;
    double hmax = 0.0;
    long long sup = 0;
#pragma unroll UK
    for (int k = 0; k < M; ++k) {
      const double h = branch == 0 ? 0.0 : (branch == 1 ? VG(k) : soft(VG(k), th));
      VSET(k, h);  // v holds h from here on (an escalation recomputes v)
      sup += (h != 0.0);
      hmax = fmax(hmax, fabs(h));
    }
    double gdl = 0.0, lmax = 0.0, dnz = 0.0;
    if (a.mode != PROJ_ALPHA0) {
      // stage h, then coalesced d = h - x (written out) and leaf g_j d_j
      if (!VS) {
#pragma unroll
        for (int k = 0; k < M; ++k) vbuf[swz<M>(tid * M + k)] = VG(k);
      }
      __syncthreads();
      mark(30);
#pragma unroll UB
      for (int i0 = 0; i0 < M; i0 += LB) {
        double xb[LB], gb[LB];
        load_batch<LB, KEEP>(xb, gb, xr, gr, x, g, i0, tid, base, lim, a.mode == PROJ_ITER);
#pragma unroll
        for (int b = 0; b < LB; ++b) {
          const int64_t j = tid + (int64_t)PT * (i0 + b);
          const int p = swz<M>((int)j);
          const double h = vbuf[p];
          double leaf = 0.0;
          bool nz = false;
          if (j < lim) {
            const int64_t gj = base + j;
            const double dj = a.mode == PROJ_PLAIN ? h : sub(h, xb[b]);
            lmax = fmax(lmax, fabs(dj));
            dout[gj] = dj;
            if (a.mode == PROJ_ITER) leaf = mul(gb[b], dj);
            nz = dj != 0.0;
          }
          vbuf[p] = leaf;
          // support bitmap of d for the sparse forward product (whole warps are in or out)
          const unsigned bits = __ballot_sync(0xffffffffu, nz);
          if (a.mode == PROJ_ITER && (tid & 31) == 0 && j < lim) {
            a.vb.dmask[(pofs + base + j) >> 5] = bits;
            dnz += (double)__popc(bits);
          }
        }
      }
      __syncthreads();
      mark(31);
      if (a.mode == PROJ_ITER) {
        if (!VS) {
#pragma unroll
          for (int k = 0; k < M; ++k) VSET(k, vbuf[swz<M>(tid * M + k)]);
        }
        gdl = run_tree<M, VS>([&](int k) { return VG(k); });
      }
    }
    double red2[5] = {gdl, lmax, hmax, (double)sup, dnz};
    const int kinds2[5] = {0, 1, 1, 3, 3};
    block_reduce<5>(red2, kinds2, sh, rp);
    mark(4);
    cluster_combine(red2, kinds2, 5, sh, cl, cs, rp);
    const double gd = red2[0], stat = red2[1], hinf = red2[2];
    const long long support = (long long)red2[3];
    mark(7);

    if (a.mode != PROJ_ITER) {
      if (rank == 0 && tid == 0) {
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
    if (stat <= sst.stationarity_tol) outcome = 0;
    else if (gd < 0.0) outcome = 1;
    else if (alpha >= cfg.alpha_max) outcome = 2;
    else outcome = 3;
    if (outcome == 3) {
      const double a10 = mul(alpha, 10.0);
      alpha = a10 < cfg.alpha_max ? a10 : cfg.alpha_max;
      continue;
    }
    if (rank == 0 && tid == 0) {
      st->out_stationarity = outcome == 2 ? first_stat : stat;
      if (outcome == 1) {
        st->dsup = (int64_t)red2[4];  // nonzeros of d: the forward product's density switch
        st->alpha_used = alpha;
        st->stat = stat;
        st->gd = gd;
        st->theta = theta;
        st->support = support;
      } else {
        st->stationary = 1;
        st->reason = L1G_STATIONARY;
        leave_run(st, STOPPED);
        l1g_iter_record& r = st->last;
        r.k = sst.k;
        r.f = sst.f;
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
  if (prof)
    for (int i = 0; i < 32; ++i) st->prof[i] = sst.prof[i];
  L1G_TL_STAMP(a.mode == PROJ_ITER && blockIdx.x == 0 && tid == 0, g_tl_proj, 14, sst.k)
  cl.sync();
}

// ---------------------------------------------------------------- host side
static int64_t pow2_at_least(int64_t v) {
  int64_t n = 1;
  while (n < v) n <<= 1;
  return n;
}

// Dynamic shared memory: [candidates] when v is in registers; [v (LS) | candidates] when v
// lives in shared memory (M >= L1G_PROJ_VS_MIN, see proj_kernel), with at most vs_cand(M)
// candidates beside v (the 1024 key bins of M >= 16 take 24 KB more static memory).
static constexpr int64_t vs_cand(int M) { return M >= 16 ? 8192 : SMEM_CAND; }
static constexpr size_t proj_dyn_bytes(int M) {
  return (M >= L1G_PROJ_VS_MIN && M <= 32) ? (size_t)(PT * M + vs_cand(M) + 1) * 8
                                           : (size_t)(SMEM_CAND + 1) * 8;
}
static void set_proj_smem(ProjPlan& pp) {
  const int M = (int)(pp.ls / PT);
  if (M >= L1G_PROJ_VS_MIN && M <= 32) {
    if (pp.cand_cap > vs_cand(M) + 1) pp.cand_cap = vs_cand(M) + 1;
    pp.smem = (size_t)(pp.ls + pp.cand_cap) * 8;
  } else {
    if (M > 32 && pp.cand_cap > SMEM_CAND + 1) pp.cand_cap = SMEM_CAND + 1;  // v is global
    pp.smem = (size_t)pp.cand_cap * 8;
  }
}

ProjPlan make_proj_plan(int64_t p_pad) {
  // small vectors: one CTA; otherwise >= 4 elements per thread spread over up to 16 CTAs
  // so the O(p) passes use enough SMs
  ProjPlan pp{};
  int64_t m = 1;
  int cs = 1;
  if (p_pad <= 8 * PT) {
    while (PT * m < p_pad) m <<= 1;
  } else {
    m = 4;
    while (PT * m * MAX_CS < p_pad) m <<= 1;
    if (m > MAX_M) throw InvalidArgument("projection: p too large for the cluster kernel");
    const int64_t need = (p_pad + PT * m - 1) / (PT * m);
    while (cs < need) cs <<= 1;
  }
  pp.cs = cs;
  pp.ls = PT * m;
  pp.cand_cap = (pp.ls > SMEM_CAND ? pp.ls : SMEM_CAND) + 1;
  set_proj_smem(pp);
  return pp;
}

// [candidates: next_pow2(p_pad) + 1 | v of M > 32 plans: 2 next_pow2(p_pad) (>= cs * ls)]
size_t proj_scratch_doubles(int64_t p_pad) {
  return (size_t)(pow2_at_least(p_pad) + 1) + (size_t)(2 * pow2_at_least(p_pad) + 2) + 64;
}

template <int M>
static void proj_launch(const ProjPlan& pp, const ProjArgs& a, cudaStream_t s, int nprob) {
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    L1G_CUDA(cudaFuncSetAttribute(proj_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)proj_dyn_bytes(M)));
    L1G_CUDA(cudaFuncSetAttribute(proj_kernel<M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pp.cs * nprob, 1, 1);
  cfg.blockDim = dim3(PT, 1, 1);
  cfg.dynamicSmemBytes = pp.smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = pp.cs;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  L1G_CUDA(cudaLaunchKernelEx(&cfg, proj_kernel<M>, a));
}

static void proj_dispatch(const ProjPlan& pp, const ProjArgs& a, cudaStream_t s, int nprob) {
  switch (pp.ls / PT) {
    case 1: proj_launch<1>(pp, a, s, nprob); break;
    case 2: proj_launch<2>(pp, a, s, nprob); break;
    case 4: proj_launch<4>(pp, a, s, nprob); break;
    case 8: proj_launch<8>(pp, a, s, nprob); break;
    case 16: proj_launch<16>(pp, a, s, nprob); break;
    case 32: proj_launch<32>(pp, a, s, nprob); break;
    case 64: proj_launch<64>(pp, a, s, nprob); break;
    case 128: proj_launch<128>(pp, a, s, nprob); break;
    case 256: proj_launch<256>(pp, a, s, nprob); break;
    case 512: proj_launch<512>(pp, a, s, nprob); break;
    default: throw InvalidArgument("projection: unsupported slice length");
  }
}

void launch_proj(const ProjPlan& pp, int mode, int64_t p, int64_t p_pad, const double* xin,
                 const double* gin, double* out, double* scratch, DevState* st,
                 const VecBufs* vb, cudaStream_t s, int nprob, int64_t scr_stride,
                 const double* rank_scal, int nranks, const int* sel, int sel_thr, int sel_mode) {
  if (nranks > 16) throw InvalidArgument("sharded solver: at most 16 ranks");
  ProjArgs a{};
  a.rank_scal = rank_scal;
  a.nranks = rank_scal ? nranks : 1;
  a.sel = sel;
  a.sel_thr = sel_thr;
  a.sel_mode = sel ? sel_mode : 0;
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
  a.bstride = nprob > 1 ? p_pad : 0;
  a.scr_stride = scr_stride;
  proj_dispatch(pp, a, s, nprob);
}

// batched runs: a cluster of `cs` CTAs per problem (1: the whole vector in one CTA)
ProjPlan make_proj_plan_single(int64_t p_pad, int cs) {
  ProjPlan pp{};
  int64_t m = 1;
  while (PT * m * cs < p_pad) m <<= 1;
  if (m > MAX_M) return make_proj_plan(p_pad);
  pp.cs = cs;
  pp.ls = PT * m;
  pp.cand_cap = (pp.ls > SMEM_CAND ? pp.ls : SMEM_CAND) + 1;
  if (cs == 1) pp.cand_cap = pp.ls + 1;
  set_proj_smem(pp);
  return pp;
}

}  // namespace l1g

#ifdef L1G_PROJ_TRACE
extern "C" int l1g_debug_prefix_trace(long long* trace192, long long* stamps520) {
  cudaMemcpyFromSymbol(trace192, g_ptrace, sizeof(long long) * 192);
  cudaMemcpyFromSymbol(stamps520, g_pstamp, sizeof(long long) * 65 * 8);
  return 0;
}
#endif

#ifdef L1G_TIMELINE
extern "C" int l1g_debug_timeline_proj(unsigned long long* out4096, int reset) {
  if (reset) {
    static unsigned long long ones[256 * 16];
    for (auto& v : ones) v = ~0ull;
    return (int)cudaMemcpyToSymbol(l1g::g_tl_proj, ones, sizeof(ones));
  }
  return (int)cudaMemcpyFromSymbol(out4096, l1g::g_tl_proj, sizeof(unsigned long long) * 256 * 16);
}
#endif
