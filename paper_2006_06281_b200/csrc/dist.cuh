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
void launch_sigma_local_sum(const double* sig_part, int blocks, double* out, const IterState* st,
                            cudaStream_t s);

}  // namespace fcpd
