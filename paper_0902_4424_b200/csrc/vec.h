// vec.h -- host launchers for vec.cu
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"

namespace l1g {

enum RedOp : int { RED_DOT = 0, RED_SQ = 1, RED_ABS = 2, RED_MAX = 3 };

void tile_rows_from_rowmajor(double* K, const GemvPlan& pl, const double* src_dev, int64_t row0,
                             int64_t rows, cudaStream_t s);
void tile_from_colmajor(double* K, const GemvPlan& pl, const double* src_dev, cudaStream_t s);
void generate_gaussian(double* K, const GemvPlan& pl, uint64_t seed, int64_t col_offset,
                       int64_t p_total, cudaStream_t s);
void generate_blur(double* K, const GemvPlan& pl, const double* taps_dev, int radius,
                   cudaStream_t s);
void scale(double* a, int64_t m, double c, cudaStream_t s);
void untile_rows(const double* K, const GemvPlan& pl, double* dst, int64_t row0, int64_t rows,
                 cudaStream_t s);
void reduce(const double* a, const double* b, int64_t m, int op, double* out, int do_sqrt,
            cudaStream_t s);
void fill(double* a, int64_t m, int64_t valid, double c, cudaStream_t s);
void div_by(const double* w, double* v, int64_t m, const double* nrm, cudaStream_t s);
void soft_threshold(const double* x, double* out, int64_t m, double t, cudaStream_t s);
void vsub(const double* a, const double* b, double* out, int64_t m, cudaStream_t s);
void lincomb(const double* a, double alpha, const double* b, double* out, int64_t m,
             cudaStream_t s);
void extrap(const double* x, const double* xprev, double coef, double* out, int64_t m,
            cudaStream_t s);
void steplength_device(l1g_sl_state* sl, const double* dots, const l1g_gp_config& cfg,
                       l1g_sl_choice* out, cudaStream_t s);
void backtrack_device(const double* in, const l1g_gp_config& cfg, double* out, cudaStream_t s);
void state_start(DevState* st, cudaStream_t s);
void rng_fill(int kind, uint64_t seed, uint32_t stream, uint64_t first, int64_t count,
              double* out, cudaStream_t s);

}  // namespace l1g
