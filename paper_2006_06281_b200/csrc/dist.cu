// dist.cu — kernels of the multi-GPU (one process per GPU, NCCL) EM path.
//
// Sharding: scene points N are split over ranks (pass 1 is
// column-local: no communication); every rank accumulates pass-2 row
// partials over its columns for all M rows, a reduce-scatter hands each rank
// the global sums of its own contiguous row shard; the M-step is row-sharded
// (z = Σ_r Q_rᵀ R_r → all-reduce K×3; V_r = Q_r g), the σ² partials are
// all-reduced, and x̃ is all-gathered for the next E-step.  Rows whose global
// mass is tiny take the exact max-shifted fallback with two collectives
// (all-reduce MAX of the row maxima, reduce-scatter of shifted sums).
//
// Row-sum layout for the collectives is AoS [M_pad][5] so each rank's rows
// are one contiguous chunk.

#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "dist.cuh"
#include "mstep.cuh"

namespace fcpd {

namespace {

__device__ __forceinline__ float sqdist_d(float4 a, float4 b) {
  const float dx = __fsub_rn(a.x, b.x);
  const float dy = __fsub_rn(a.y, b.y);
  const float dz = __fsub_rn(a.z, b.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}
__device__ __forceinline__ float4 scale_d(float4 p, float s) {
  return make_float4(__fmul_rn(p.x, s), __fmul_rn(p.y, s), __fmul_rn(p.z, s), p.w);
}
}  // namespace

// part [splits][5][M] → out [M_pad][5] (pad rows zero), 8 lanes per row.
__device__ __forceinline__ void finalize_own(int64_t i, int64_t mr, double log2p1, double s0,
                                             double sy0, double sy1, double sy2, double sv,
                                             const double* __restrict__ xt64_own, double s,
                                             const DistRowOut& o, const YStats& ys,
                                             IterState* st) {
  const double x0 = xt64_own[i], x1 = xt64_own[mr + i], x2 = xt64_own[2 * mr + i];
  double p0, p1, p2, var;
  int deg = 0;
  if (log2p1 < kLog2DegenerateRow) {
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
  o.ptilde_y[i] = p0;
  o.ptilde_y[mr + i] = p1;
  o.ptilde_y[2 * mr + i] = p2;
  o.var[i] = var;
  o.log2p1[i] = log2p1;
  o.degenerate[i] = deg;
  o.resid4[i] = make_float4(static_cast<float>(p0 - o.x0_own[i]),
                            static_cast<float>(p1 - o.x0_own[mr + i]),
                            static_cast<float>(p2 - o.x0_own[2 * mr + i]), 0.f);
}

// Own rows: global sums → finalize, or flag (mask) for the exact fallback.
__global__ void row_finalize_own_kernel(const double* __restrict__ sums_own, int64_t mr,
                                        int64_t m_valid_own, int64_t n_global,
                                        const double* __restrict__ xt64_own, DistRowOut o,
                                        YStats ys, int32_t* __restrict__ mask_own,
                                        IterState* st) {
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= mr) return;
  if (i >= m_valid_own) {  // padding rows: never flagged, inert residual
    mask_own[i] = 0;
    o.resid4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const double* a = sums_own + i * 5;
  const bool flagged = !(a[0] >= static_cast<double>(n_global) * 0x1p-76);
  mask_own[i] = flagged ? 1 : 0;
  if (flagged) {
    // the exact fallback fills this row later; until then it adds nothing
    // to z (its contribution is the z correction), and it is counted for
    // the group-wide "any row flagged" test
    o.resid4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    atomicAdd(&st->flag_count[1], 1);
    return;
  }
  const double s = sqrt(kLog2e / (2.0 * st->sigma2_e));
  finalize_own(i, mr, log2(a[0]), a[0], a[1], a[2], a[3], a[4], xt64_own, s, o, ys, st);
}

// Flagged rows (any rank): max over this rank's columns of L = b − t.
__global__ void fallback_max_kernel(const int32_t* __restrict__ mask_all, int64_t m_pad,
                                    const float4* __restrict__ xt4, const float4* __restrict__ y4b,
                                    int64_t n_local, float* __restrict__ out_max,
                                    const IterState* __restrict__ st) {
  if (!st->active) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(blockDim.x >> 5) * gridDim.x;
  const float s = st->sx;
  for (int64_t row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m_pad;
       row += warps) {
    float lmax = -INFINITY;
    if (mask_all[row]) {
      const float4 xv = scale_d(xt4[row], s);
      for (int64_t j = lane; j < n_local; j += 32) {
        const float4 yv = scale_d(y4b[j], s);
        lmax = fmaxf(lmax, yv.w - sqdist_d(yv, xv));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if (lane == 0) out_max[row] = lmax;
  }
}

// Flagged rows: fp64 sums of 2^{L − gmax} over this rank's columns.
__global__ void fallback_sum_kernel(const int32_t* __restrict__ mask_all, int64_t m_pad,
                                    const float* __restrict__ gmax, const float4* __restrict__ xt4,
                                    const float4* __restrict__ y4b, int64_t n_local,
                                    double* __restrict__ out, const IterState* __restrict__ st) {
  if (!st->active) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(blockDim.x >> 5) * gridDim.x;
  const float s = st->sx;
  for (int64_t row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m_pad;
       row += warps) {
    double a0 = 0, ax = 0, ay = 0, az = 0, av = 0;
    const float lmax = gmax[row];
    if (mask_all[row] && lmax > -INFINITY) {
      const float4 xv = scale_d(xt4[row], s);
      for (int64_t j = lane; j < n_local; j += 32) {
        const float4 yv = scale_d(y4b[j], s);
        const float t = sqdist_d(yv, xv);
        const double w = exp2(static_cast<double>(yv.w - t) - static_cast<double>(lmax));
        a0 += w;
        ax += w * yv.x;
        ay += w * yv.y;
        az += w * yv.z;
        av += w * t;
      }
      a0 = warp_sum(a0);
      ax = warp_sum(ax);
      ay = warp_sum(ay);
      az = warp_sum(az);
      av = warp_sum(av);
    }
    if (lane == 0) {
      double* o = out + row * 5;
      o[0] = a0;
      o[1] = ax;
      o[2] = ay;
      o[3] = az;
      o[4] = av;
    }
  }
}

__global__ void fallback_finalize_own_kernel(const double* __restrict__ fsum_own,
                                             const float* __restrict__ gmax_own,
                                             const int32_t* __restrict__ mask_own, int64_t mr,
                                             const double* __restrict__ xt64_own, DistRowOut o,
                                             YStats ys, IterState* st) {
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= mr || !mask_own[i]) return;
  const double* a = fsum_own + i * 5;
  const double log2p1 = a[0] > 0 ? static_cast<double>(gmax_own[i]) + log2(a[0]) : -INFINITY;
  const double s = sqrt(kLog2e / (2.0 * st->sigma2_e));
  finalize_own(i, mr, log2p1, a[0], a[1], a[2], a[3], a[4], xt64_own, s, o, ys, st);
}

// σ² block partials → one local double (fixed order).
__global__ void sigma_local_sum_kernel(const double* __restrict__ sig_part, int blocks,
                                       double* __restrict__ out, float4* pack_dst,
                                       const IterState* st) {
  if (!st->active) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < blocks; b += blockDim.x) s += sig_part[b];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) t += red[w];
    if (out) out[0] = t;
    if (pack_dst) {  // the rank's σ² partial rides in the unused .w of its first two x̃ rows
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(t));
      pack_dst[0].w = __uint_as_float(static_cast<unsigned>(b & 0xffffffffull));
      pack_dst[1].w = __uint_as_float(static_cast<unsigned>(b >> 32));
    }
  }
}

// σ² after the x̃ all-gather: the G rank partials (packed by
// sigma_local_sum_kernel into .w of rows r·M_r, r·M_r + 1) summed in rank
// order — the same value on every rank — then the iteration's last step.
__global__ void sigma_final_gathered_kernel(const float4* __restrict__ xt4, int64_t mr, int world,
                                            int64_t m_global, int d, int early_stop,
                                            double* __restrict__ trace, IterState* st,
                                            uint64_t* stamps) {
  if (!st->active) return;
  double tot = 0.0;
  for (int r = 0; r < world; ++r) {
    const unsigned lo = __float_as_uint(xt4[r * mr].w), hi = __float_as_uint(xt4[r * mr + 1].w);
    tot += __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) |
                                                       lo));
  }
  finish_iteration_sigma(st, tot, m_global, d, early_stop, trace, stamps);
}

// z correction of the rows the exact fallback filled: Σ over flagged own
// rows of Qᵀ_own[k][i]·R_i (one block per eigenvector, fixed-order tree).
__global__ void zcorr_kernel(const float* __restrict__ qt_own, int64_t ld, int64_t k,
                             const int32_t* __restrict__ mask_own, const float4* __restrict__ resid4,
                             int64_t mr, double* __restrict__ zc, const IterState* st) {
  if (!st->active) return;
  __shared__ double red[3][32];
  const int64_t kk = blockIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t i = threadIdx.x; i < mr; i += blockDim.x) {
    if (!mask_own[i]) continue;
    const double q = qt_own[kk * ld + i];
    const float4 r = resid4[i];
    a0 += q * r.x;
    a1 += q * r.y;
    a2 += q * r.z;
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  a2 = warp_sum(a2);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[0][w] = a0, red[1][w] = a1, red[2][w] = a2;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s[3] = {0.0, 0.0, 0.0};
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s[c] += red[c][i];
  zc[kk] = s[0];
  zc[k + kk] = s[1];
  zc[2 * k + kk] = s[2];
}

__global__ void zadd_kernel(double* __restrict__ z, const double* __restrict__ zc, int64_t count,
                            const IterState* st) {
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) z[i] += zc[i];
}

// the group-wide flagged-row count rides in z[3K] of the z all-reduce:
// run the fallback exchange (a conditional graph node) only when nonzero
__global__ void set_fallback_cond_kernel(cudaGraphConditionalHandle h,
                                         const double* __restrict__ zfull, int64_t k,
                                         const IterState* st) {
  cudaGraphSetConditional(h, st->active && zfull[3 * k] > 0.5 ? 1u : 0u);
}

// rowdot_reduce's z all-reduce payload gets the local flagged-row count
__global__ void put_flag_count_kernel(double* __restrict__ zfull, int64_t k, const IterState* st) {
  zfull[3 * k] = st->active ? static_cast<double>(st->flag_count[1]) : 0.0;
}

// ------------------------------------------------------------------ launchers

void launch_row_finalize_own(const double* sums_own, int64_t mr, int64_t m_valid_own,
                             int64_t n_global, const double* xt64_own, const DistRowOut& o,
                             const YStats& ys, int32_t* mask_own, IterState* st, cudaStream_t s) {
  row_finalize_own_kernel<<<ceil_div(mr, 256), 256, 0, s>>>(sums_own, mr, m_valid_own, n_global,
                                                            xt64_own, o, ys, mask_own, st);
  FCPD_LAUNCH_CHECK();
}
void launch_fallback_max(const int32_t* mask_all, int64_t m_pad, const float4* xt4,
                         const float4* y4b, int64_t n_local, float* out_max, const IterState* st,
                         cudaStream_t s) {
  fallback_max_kernel<<<148, 256, 0, s>>>(mask_all, m_pad, xt4, y4b, n_local, out_max, st);
  FCPD_LAUNCH_CHECK();
}
void launch_fallback_sum(const int32_t* mask_all, int64_t m_pad, const float* gmax,
                         const float4* xt4, const float4* y4b, int64_t n_local, double* out,
                         const IterState* st, cudaStream_t s) {
  fallback_sum_kernel<<<148, 256, 0, s>>>(mask_all, m_pad, gmax, xt4, y4b, n_local, out, st);
  FCPD_LAUNCH_CHECK();
}
void launch_fallback_finalize_own(const double* fsum_own, const float* gmax_own,
                                  const int32_t* mask_own, int64_t mr, const double* xt64_own,
                                  const DistRowOut& o, const YStats& ys, IterState* st,
                                  cudaStream_t s) {
  fallback_finalize_own_kernel<<<ceil_div(mr, 256), 256, 0, s>>>(fsum_own, gmax_own, mask_own, mr,
                                                                 xt64_own, o, ys, st);
  FCPD_LAUNCH_CHECK();
}
void launch_sigma_local_sum(const double* sig_part, int blocks, double* out, float4* pack_dst,
                            const IterState* st, cudaStream_t s) {
  sigma_local_sum_kernel<<<1, 256, 0, s>>>(sig_part, blocks, out, pack_dst, st);
  FCPD_LAUNCH_CHECK();
}

void launch_sigma_final_gathered(const float4* xt4, int64_t mr, int world, int64_t m_global, int d,
                                 int early_stop, double* trace, IterState* st, uint64_t* stamps,
                                 cudaStream_t s) {
  sigma_final_gathered_kernel<<<1, 1, 0, s>>>(xt4, mr, world, m_global, d, early_stop, trace, st,
                                              stamps);
  FCPD_LAUNCH_CHECK();
}

void launch_zcorr(const float* qt_own, int64_t ld, int64_t k, const int32_t* mask_own,
                  const float4* resid4, int64_t mr, double* zc, const IterState* st, cudaStream_t s) {
  zcorr_kernel<<<static_cast<unsigned>(k), 256, 0, s>>>(qt_own, ld, k, mask_own, resid4, mr, zc, st);
  FCPD_LAUNCH_CHECK();
}

void launch_zadd(double* z, const double* zc, int64_t count, const IterState* st, cudaStream_t s) {
  zadd_kernel<<<ceil_div(count, 256), 256, 0, s>>>(z, zc, count, st);
  FCPD_LAUNCH_CHECK();
}

void launch_set_fallback_cond(cudaGraphConditionalHandle h, const double* zfull, int64_t k,
                              const IterState* st, cudaStream_t s) {
  set_fallback_cond_kernel<<<1, 1, 0, s>>>(h, zfull, k, st);
  FCPD_LAUNCH_CHECK();
}

void launch_put_flag_count(double* zfull, int64_t k, const IterState* st, cudaStream_t s) {
  put_flag_count_kernel<<<1, 1, 0, s>>>(zfull, k, st);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
