// mstep.cuh — M-step / transform / σ² launch interface (see mstep.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace fcpd {

struct ColsumPlan {
  int64_t cols4 = 0;
  int col_blocks = 0;
  int row_blocks = 0;
  int64_t rows_per_block = 0;
};

ColsumPlan make_colsum_plan(int64_t rows, int64_t cols, int sm_count);

// part[rb][d][c] (d<3, leading dimension part_ld ≥ 4·cols4) =
//   Σ_{r∈rb} A[r][c]·v[r].d ;  A row-major fp32 with lda % 4 == 0.
void launch_colsum(const ColsumPlan& p, const float* A, int64_t lda, int64_t rows,
                   const float4* v, double* part, int64_t part_ld, const IterState* st,
                   uint64_t* stamps, int stamp_slot, cudaStream_t stream);

void launch_zreduce(const double* part, int blocks, int64_t k, int64_t part_ld,
                    const double* lam, const double* lam_num, double lambda_reg, double* coef,
                    float4* g4, IterState* st, cudaStream_t stream);

void launch_transform_sigma(const double* part, int blocks, int64_t m, int64_t part_ld,
                            const double* x0, double* xt64, double* xt_prev, float4* xt4,
                            const double* ptilde_y, const double* var, double* sig_part,
                            int d, int early_stop, double* trace, IterState* st,
                            uint64_t* stamps, cudaStream_t stream);

}  // namespace fcpd

namespace fcpd {
void launch_vreduce_add(const double* part, int blocks, int64_t m, int64_t part_ld,
                        const double* x0, int d, double* out, cudaStream_t stream);
}  // namespace fcpd
