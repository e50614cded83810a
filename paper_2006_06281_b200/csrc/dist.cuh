// dist.cuh — multi-GPU EM kernels (see dist.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "estep.cuh"

namespace fcpd {

// Own-row outputs of the distributed E-step (local SoA arrays of M_r rows).
struct DistRowOut {
  double* ptilde_y;
  double* var;
  double* log2p1;
  int32_t* degenerate;
  float4* resid4;
  const double* x0_own;
};

void launch_row_finalize_own(const double* sums_own, int64_t mr, int64_t m_valid_own,
                             int64_t n_global, const double* xt64_own, const DistRowOut& o,
                             const YStats& ys, int32_t* mask_own, IterState* st, cudaStream_t s);
void launch_fallback_max(const int32_t* mask_all, int64_t m_pad, const float4* xt4,
                         const float4* y4b, int64_t n_local, float* out_max, const IterState* st,
                         cudaStream_t s);
void launch_fallback_sum(const int32_t* mask_all, int64_t m_pad, const float* gmax,
                         const float4* xt4, const float4* y4b, int64_t n_local, double* out,
                         const IterState* st, cudaStream_t s);
void launch_fallback_finalize_own(const double* fsum_own, const float* gmax_own,
                                  const int32_t* mask_own, int64_t mr, const double* xt64_own,
                                  const DistRowOut& o, const YStats& ys, IterState* st,
                                  cudaStream_t s);
// σ² partial of the own rows → out and/or packed into pack_dst[0..1].w
void launch_sigma_local_sum(const double* sig_part, int blocks, double* out, float4* pack_dst,
                            const IterState* st, cudaStream_t s);
// after the x̃ all-gather: Σ of the G packed partials (rank order) → σ², trace
void launch_sigma_final_gathered(const float4* xt4, int64_t mr, int world, int64_t m_global, int d,
                                 int early_stop, double* trace, IterState* st, uint64_t* stamps,
                                 cudaStream_t s);
// z correction from the rows the fallback filled, and its addition
void launch_zcorr(const float* qt_own, int64_t ld, int64_t k, const int32_t* mask_own,
                  const float4* resid4, int64_t mr, double* zc, const IterState* st, cudaStream_t s);
void launch_zadd(double* z, const double* zc, int64_t count, const IterState* st, cudaStream_t s);
// conditional-node predicate: any row flagged group-wide (z[3K] after the all-reduce)
void launch_set_fallback_cond(cudaGraphConditionalHandle h, const double* zfull, int64_t k,
                              const IterState* st, cudaStream_t s);
void launch_put_flag_count(double* zfull, int64_t k, const IterState* st, cudaStream_t s);

}  // namespace fcpd
