// engine.h -- internal structures shared by the host runtime and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/l1g.h"

namespace l1g {

struct CudaError : std::runtime_error {
  CudaError(cudaError_t e, const char* call, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + call +
                           " at " + file + ":" + std::to_string(line)) {}
};
struct InvalidArgument : std::invalid_argument {
  explicit InvalidArgument(const std::string& m) : std::invalid_argument(m) {}
};
struct RuntimeFailure : std::runtime_error {
  explicit RuntimeFailure(const std::string& m) : std::runtime_error(m) {}
};
// an iteration callback returned nonzero (L1G_ECANCELED)
struct Cancelled : std::runtime_error {
  Cancelled() : std::runtime_error("iteration callback stopped the run") {}
};

constexpr int kMaxHist = 64;

enum Status : int { RUNNING = 0, STOPPED = 1, FAILED = 2 };
enum Failure : int { FAIL_NONE = 0, FAIL_BACKTRACK = 1 };

// Device-resident scalar state of one GPSS run (GpIterationState + SteplengthState +
// the gpss_solve loop variables, gpss.hpp:31-36, :89-98; gpss.cpp:226-231).
struct DevState {
  // configuration
  l1g_gp_config cfg;
  double rho;
  double stationarity_tol, objective_tol, max_seconds;
  int64_t max_iterations, max_matvecs;
  int single_step;  // 1: gp_iterate semantics (no budget checks, no objective_tol)
  // run control
  int status, reason, failure, cur;
  uint64_t t_start;
  // GP state
  int64_t k, matvecs;
  double f, f_prev;
  double fh[kMaxHist];
  int fh_len;
  double tau;
  double a2h[kMaxHist + 2];
  int a2_len;
  double alpha0;
  int stationary;
  double out_stationarity;
  // secant dots of the last step (s = x_k - x_{k-1}, z = g_k - g_{k-1})
  double sz, ss, zz;
  // per-iteration values
  l1g_sl_choice choice;
  double alpha_used, stat, gd, theta, f_max, step, f_new, a, b;
  int32_t halvings;
  int64_t support;
  int64_t dsup;  // nonzeros of the last direction d (the forward product's support columns)
  l1g_iter_record last;  // record of the last completed (or stationary) iteration
  // telemetry
  l1g_iter_record* trace;
  int64_t trace_cap;
  // init checks
  double x0_l1;
  double h_inf;  // alpha0 projection inf-norm
  // projection phase profile (SM cycles of CTA 0 / event counts), see project.cu
  double prof[32];
  // batched runs: live-problem counter, decremented when this problem stops (steps.cuh)
  int* nrun;
};
static_assert(sizeof(DevState) % 8 == 0, "DevState is copied as 8-byte words");

// GEMV launch plan for one operator
struct GemvPlan {
  int64_t n, p, n_pad, p_pad, nrb, ncb;
  // forward: tasks = row group (128 rows) x column range (fwd_stages * 64 columns)
  int fwd_stages, nrg, ncr;
  // adjoint: tasks = column group (256 columns) x row range (adj_blocks * 32 rows)
  int adj_blocks, ncg, nrr;
  // sparse forward (support columns only): column ranges of sp_tiles * 64 columns
  int sp_tiles, sp_ncr;
  // the sparse forward switches to the dense TMA stream (fwd_kernel) on the device when d
  // has at least this many nonzeros (measured crossover)
  int64_t dense_min;
  int grid;
};

struct Ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  // scratch for host-vector entry points
  double* scratch = nullptr;
  size_t scratch_len = 0;
  DevState* scratch_state = nullptr;
  double* scratch_d = nullptr;  // small device scalars
};

struct Op {
  Ctx* ctx = nullptr;
  GemvPlan plan{};
  double* K = nullptr;  // tiled
};

// per-run scratch of the two GEMV kernels (one per solver / per op for generic applies)
struct Workspace {
  double* fwd_part = nullptr;    // ncr * n_pad
  double* adj_part = nullptr;    // nrr * p_pad
  double* grpsum = nullptr;      // max(nrg*2, ncg*3)
  unsigned* counters = nullptr;  // [nrg + ncg + 2], zero between launches
};

// projection plan (cluster of cs CTAs, each holding an aligned slice of ls elements)
struct ProjPlan {
  int cs;
  int64_t ls;
  int64_t cand_cap;  // candidates sortable in CTA 0 shared memory
  size_t smem;
};

enum FwdMode : int { FWD_APPLY = 0, FWD_INIT = 1, FWD_ITER = 2 };
enum AdjMode : int { ADJ_APPLY = 0, ADJ_INIT = 1, ADJ_ITER = 2 };
enum ProjMode : int { PROJ_PLAIN = 0, PROJ_ALPHA0 = 1, PROJ_ITER = 2 };

struct VecBufs {
  double* x[2];
  double* g[2];
  double* r[2];
  double* d;
  double* kd;
  const double* y;
  uint32_t* dmask;  // support bitmap of d (bit j of word j/32), written by proj_kernel
};

// batched-RHS products on the FP64 tensor cores (dmma.cu)
struct BatchPlan {
  int B, Bp;                 // problems, padded to the CTA width (128)
  int fwd_splits, fwd_per;   // column blocks per split of the forward reduction
  int adj_splits, adj_per;   // row blocks per split of the adjoint reduction
  int wide;                  // 1: the 16-warp 128x128 product kernels (dmma.cu), 0: 8-warp
};
struct BGemmArgs {
  const double* K;
  int64_t ncb, nrb;
  const double* V;   // forward: D [Bp][p_pad]; adjoint: R [Bp][n_pad]
  int64_t vstride;
  double* part;      // [splits][Bp][ostride]
  int64_t pslab, ostride;
  int per_split, nblocks;
  int nx, ny, nz;  // persistent products: work items (tiles x splits x problem blocks)
  // live-problem compaction (producer-warp products): column j of the product is problem
  // active[j], j < *nact; problem blocks, 32-problem warp groups and 8-problem tiles past
  // *nact are skipped.  nullptr: every problem, in place.
  const int* active;
  const int* nact;
  int nb;  // problems in the batch: *nact == nb means all live (active[] is the identity)
  int tail;  // a bws_tail_kernel launch follows: it takes the launch when *nact <= 8
};
struct BFinArgs {  // batched finishes (dmma.cu): problem b's vectors at b * ostride
  int mode, B, splits;
  const double* part;
  int64_t pslab, ostride;
  double* vout;
  VecBufs vb;
  DevState* st;
  unsigned* counters;
  double* grpsum;
  int64_t grp_stride;
};
void launch_bfin(const BFinArgs& a, bool adjoint, int64_t len_pad, cudaStream_t s);
void launch_brupdate(const BFinArgs& a, double* rn, cudaStream_t s);
BatchPlan make_batch_plan(const GemvPlan& pl, int B, int sm_count);
void launch_bfwd(const Op& op, const BatchPlan& bp, const double* D, double* part, cudaStream_t s,
                 const int* active = nullptr, const int* nact = nullptr);
void launch_badj(const Op& op, const BatchPlan& bp, const double* R, double* part, cudaStream_t s,
                 const int* active = nullptr, const int* nact = nullptr);
bool batch_tail_kernels();
void launch_bcompact(const DevState* st, int B, int* active, int* nact, cudaStream_t s);

// small problems (small.cu): the whole step after the projection as one cluster kernel
bool small_iter_fits(const GemvPlan& pl);
void launch_small_iter(const Op& op, const VecBufs* vb, DevState* st, cudaStream_t s);

// host launchers (gemv.cu, project.cu)
GemvPlan make_plan(int64_t n, int64_t p, int sm_count);
void launch_fwd(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout, const VecBufs* vb,
                DevState* st, cudaStream_t s, bool sparse = false, bool dense_switch = false);
void launch_fwd_init_zero(const Op& op, const Workspace& ws, const VecBufs* vb, DevState* st,
                          cudaStream_t s);
void launch_adj(const Op& op, const Workspace& ws, int mode, const double* vin, double* vout, const VecBufs* vb,
                DevState* st, cudaStream_t s, double* pack = nullptr);
// scalars per rank in a shard's allgather packet: s'z, s's, z'z subtree values, clock
constexpr int SHARD_SCAL = 8;
// column-sharded runs: the shard's tree values of K d (n_pad) and the combination of the
// gathered rank values with the fused epilogue of `mode`
void launch_fwd_part(const Op& op, const Workspace& ws, const double* vin, const uint32_t* dmask,
                     bool sparse, double* out, DevState* st, cudaStream_t s);
void launch_fwd_combine(const Op& op, const Workspace& ws, int mode, const double* recv, int nr,
                        const VecBufs* vb, DevState* st, cudaStream_t s);
ProjPlan make_proj_plan(int64_t p_pad);
// rank_scal (sharded runs): the ranks' packet scalars [nranks][SHARD_SCAL]; the projection
// joins the secant dots over the ranks and takes the budget clock from them
void launch_proj(const ProjPlan& pp, int mode, int64_t p, int64_t p_pad, const double* xin,
                 const double* gin, double* out, double* scratch, DevState* st,
                 const VecBufs* vb, cudaStream_t s, int nprob = 1, int64_t scr_stride = 0,
                 const double* rank_scal = nullptr, int nranks = 1, const int* sel = nullptr,
                 int sel_thr = 0, int sel_mode = 0);
ProjPlan make_proj_plan_single(int64_t p_pad, int cs = 1);
size_t proj_scratch_doubles(int64_t p_pad);

}  // namespace l1g
