// estep_device.cuh — E-step device helpers shared by the pass kernels
// (estep.cu) and the one-kernel small-problem iteration (mstep_fused.cu).
#pragma once

#include "common.cuh"
#include "estep.cuh"

namespace fcpd {

// the difference-form pair term t = ‖a − b‖² (scaled frame), as the pass
// kernels' difference path and the exact fallbacks
__device__ __forceinline__ float sqdist(float4 a, float4 b) {
  const float dx = __fsub_rn(a.x, b.x);
  const float dy = __fsub_rn(a.y, b.y);
  const float dz = __fsub_rn(a.z, b.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// coordinates into the scaled frame (x' = s·x); .w (b_n) passes through
__device__ __forceinline__ float4 scale_pt(float4 p, float s) {
  return make_float4(__fmul_rn(p.x, s), __fmul_rn(p.y, s), __fmul_rn(p.z, s), p.w);
}

__device__ __forceinline__ double derived_scale(const IterState* st) {
  return sqrt(kLog2e / (2.0 * st->sigma2_e));
}

// ---------------------------------------------------------------------------
// Row finalisation shared by the pass-2 block fix-up and the fallback.
__device__ __forceinline__ void finalize_row(int64_t row, int64_t m, double log2p1, double s0,
                                             double sy0, double sy1, double sy2, double sv,
                                             const double* __restrict__ xt64, double s,
                                             const RowOut& out, const YStats& ys,
                                             IterState* st) {
  const double x0 = xt64[row], x1 = xt64[m + row], x2 = xt64[2 * m + row];
  double p0, p1, p2, var;
  int deg = 0;
  if (log2p1 < kLog2DegenerateRow) {  // uniform row, correspondence.hpp:89-91
    deg = 1;
    p0 = ys.mean[0];
    p1 = ys.mean[1];
    p2 = ys.mean[2];
    var = ys.sq_mean - 2.0 * (x0 * p0 + x1 * p1 + x2 * p2) + (x0 * x0 + x1 * x1 + x2 * x2);
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->degenerate_rows), 1ull);
  } else {
    const double inv = 1.0 / (s0 * s);
    p0 = sy0 * inv;
    p1 = sy1 * inv;
    p2 = sy2 * inv;
    var = sv / (s0 * s * s);
  }
  out.ptilde_y[row] = p0;
  out.ptilde_y[m + row] = p1;
  out.ptilde_y[2 * m + row] = p2;
  out.var[row] = var;
  out.log2p1[row] = log2p1;
  out.degenerate[row] = deg;
  if (out.resid4) {
    // R = P̃Y − X (registration.hpp:136), fp32 for the Q product
    const double* X = out.x0;
    out.resid4[row] = make_float4(static_cast<float>(p0 - X[row]),
                                  static_cast<float>(p1 - X[m + row]),
                                  static_cast<float>(p2 - X[2 * m + row]), 0.f);
  }
}

}  // namespace fcpd
