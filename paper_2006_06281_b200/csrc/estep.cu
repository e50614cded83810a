// estep.cu — fused, non-materialising Fast-CPD E-step for sm_100a.
//
// Restates correspondence.hpp:35-105 (posterior → enforce_row_constraint →
// estimated_targets) and the per-row terms of update_sigma2
// (solvers.hpp:160-176) without ever forming the M×N posterior P.
//
// Notation (all in log2 units): with s = sqrt(log2e / (2σ²)), scaled points
// x' = s·x̃, y' = s·y, and t_mn = ‖y'_n − x'_m‖², the reference logit is
// e_mn = −t_mn·ln2.  Then
//   pass 1 (per scene column n, over all m):
//        b_n = −log2( Σ_m 2^{−t_mn} + [ω>0]·2^{log2 c} )
//   pass 2 (per model row m, over all n): L_mn = b_n − t_mn = log2 P_mn ≤ 0,
//        S0 = Σ_n 2^{L}, Sy = Σ_n 2^{L}·y'_n, SV = Σ_n 2^{L}·t_mn
//   so P1_m = S0, (P̃Y)_m = Sy/(s·S0), Σ_n P̃_mn‖y_n − x̃_m‖² = SV/(s²·S0).
//
// Because every term is ≤ 1 (t ≥ 0 in pass 1, L ≤ 0 in pass 2) neither pass
// needs a running max: the fast path is one ex2 (MUFU) per pair per pass.
// A column/row whose total mass is so small that fp32 flush-to-zero could
// cost more than 2^-50 relative is flagged and recomputed exactly (max-
// shifted, fp64 accumulation) by the fallback kernels; this also yields the
// reference's degenerate-row rule (row mass < 1e-300 → uniform row,
// correspondence.hpp:89-91) bit-for-bit in the decision.
//
// Work split: pass 1 tiles columns over threads (CPT per thread) and splits
// M over gridDim.y; pass 2 tiles rows over threads (RPT per thread) and
// splits N over gridDim.y.  Partials are fp64 per (split, column|row) and
// are reduced in a fixed order, so results are bitwise reproducible.

#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "estep.cuh"

namespace fcpd {

namespace {

constexpr int kTile = 256;       // points staged in shared memory per step
constexpr float kPadCoord = 3.0e18f;  // padding point: t ≈ 1e37, 2^-t = 0

__device__ __forceinline__ float sqdist(float4 a, float4 b) {
  // identical operation order in both passes (bitwise-equal t_mn)
  const float dx = __fsub_rn(a.x, b.x);
  const float dy = __fsub_rn(a.y, b.y);
  const float dz = __fsub_rn(a.z, b.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

__device__ __forceinline__ float4 scale_pt(float4 p, float s) {
  return make_float4(__fmul_rn(p.x, s), __fmul_rn(p.y, s), __fmul_rn(p.z, s), p.w);
}

__device__ __forceinline__ double derived_scale(const IterState* st) {
  return sqrt(kLog2e / (2.0 * st->sigma2_e));
}

}  // namespace

// ---------------------------------------------------------------------------
// Iteration prologue: σ² floor + clamp count (correspondence.hpp:43-47,
// registration.hpp:122), coordinate scale, outlier constant (:61-66).
__global__ void estep_prologue_kernel(IterState* st, int64_t m, int64_t n, int d,
                                      double omega, int32_t* flags_count, uint64_t* stamps) {
  if (!st->active) return;
  if (stamps) stamps[4 * st->iter + 0] = globaltimer();
  flags_count[0] = 0;
  flags_count[1] = 0;
  double s2 = st->sigma2;
  if (s2 < kSigma2Floor) {
    s2 = kSigma2Floor;
    st->sigma2_clamps += 1;
  }
  st->sigma2_e = s2;
  st->sx = static_cast<float>(sqrt(kLog2e / (2.0 * s2)));
  if (omega > 0.0) {
    const double log_c = 0.5 * d * log(2.0 * M_PI * s2) + log(omega / (1.0 - omega)) +
                         log(static_cast<double>(m) / static_cast<double>(n));
    st->log2c = log_c * kLog2e;
  } else {
    st->log2c = -INFINITY;
  }
}

// ---------------------------------------------------------------------------
// Pass 1: per-column partial sums Σ_m 2^{−t_mn} over one M-split.
template <int CPT>
__global__ void __launch_bounds__(128)
    estep_col_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4,
                     int64_t n, int64_t m_per_split, const IterState* __restrict__ st,
                     double* __restrict__ part) {
  if (!st->active) return;
  __shared__ float4 xs[kTile];
  const float s = st->sx;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * (128 * CPT) + threadIdx.x;
  float4 yv[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int64_t col = col0 + c * 128;
    yv[c] = col < n ? scale_pt(y4[col], s) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t m_begin = static_cast<int64_t>(blockIdx.y) * m_per_split;
  const int64_t m_end = min(m, m_begin + m_per_split);
  double dsum[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) dsum[c] = 0.0;

  for (int64_t base = m_begin; base < m_end; base += kTile) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), m_end - base));
    __syncthreads();
    for (int i = threadIdx.x; i < kTile; i += 128)
      xs[i] = i < cnt ? scale_pt(xt4[base + i], s)
                      : make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
    __syncthreads();
    float fsum[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) fsum[c] = 0.f;
    const int cnt8 = (cnt + 7) & ~7;
    for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 xv = xs[j + u];
#pragma unroll
        for (int c = 0; c < CPT; ++c) fsum[c] += ex2_approx(-sqdist(yv[c], xv));
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) dsum[c] += static_cast<double>(fsum[c]);
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int64_t col = col0 + c * 128;
    if (col < n) part[static_cast<int64_t>(blockIdx.y) * n + col] = dsum[c];
  }
}

// Pass 1 combine: fixed-order sum over splits; column normaliser b_n.
// Flags columns whose mass is too small for the flush-to-zero fast path.
__global__ void estep_col_combine_kernel(const double* __restrict__ part, int splits, int64_t m,
                                         int64_t n, float4* __restrict__ y4b,
                                         double* __restrict__ b2_out, double* __restrict__ pt1,
                                         int32_t* __restrict__ flag_list,
                                         int32_t* __restrict__ flag_count,
                                         const IterState* __restrict__ st) {
  if (!st->active) return;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double sm = 0.0;
  for (int s = 0; s < splits; ++s) sm += part[static_cast<int64_t>(s) * n + col];
  const double log2c = st->log2c;
  const double c = exp2(log2c);  // 0 when ω = 0
  const double total = sm + c;
  // flushed terms are < 2^-126 each: ≤ M·2^-126 in total; need ≤ 2^-50·total
  const bool flagged = !(total >= static_cast<double>(m) * 0x1p-76);
  if (flagged) {
    const int slot = atomicAdd(flag_count, 1);
    flag_list[slot] = static_cast<int32_t>(col);
    return;  // fallback writes b2 / pt1
  }
  const double b2 = -log2(total);
  b2_out[col] = b2;
  y4b[col].w = static_cast<float>(b2);
  if (pt1) pt1[col] = sm / total;
}

// Exact column normaliser for flagged columns: warp per column, max-shifted
// log-sum-exp over all m in the same fp32 t_mn, fp64 accumulation.
__global__ void estep_col_fallback_kernel(const float4* __restrict__ xt4, int64_t m,
                                          float4* __restrict__ y4b, double* __restrict__ b2_out,
                                          double* __restrict__ pt1,
                                          const int32_t* __restrict__ flag_list,
                                          const int32_t* __restrict__ flag_count,
                                          const IterState* __restrict__ st) {
  if (!st->active) return;
  const int count = *flag_count;
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  const float s = st->sx;
  const double log2c = st->log2c;
  for (int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count; w += warps) {
    const int64_t col = flag_list[w];
    const float4 yv = scale_pt(y4b[col], s);
    float tmin = INFINITY;
    for (int64_t i = lane; i < m; i += 32) tmin = fminf(tmin, sqdist(yv, scale_pt(xt4[i], s)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    // shift: reference max(max_m e, log_c) (correspondence.hpp:70-71)
    double shift = -static_cast<double>(tmin);
    if (log2c > shift) shift = log2c;
    double acc = 0.0;
    for (int64_t i = lane; i < m; i += 32) {
      const float t = sqdist(yv, scale_pt(xt4[i], s));
      acc += exp2(-static_cast<double>(t) - shift);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const double c = log2c > -INFINITY ? exp2(log2c - shift) : 0.0;
      const double b2 = -(shift + log2(acc + c));
      b2_out[col] = b2;
      y4b[col].w = static_cast<float>(b2);
      if (pt1) pt1[col] = acc / (acc + c);
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 2: per-row partial sums over one N-split: S0, Sy (3), SV.
template <int RPT>
__global__ void __launch_bounds__(128)
    estep_row_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4b,
                     int64_t n, int64_t n_per_split, const IterState* __restrict__ st,
                     double* __restrict__ part /* [split][5][m] */) {
  if (!st->active) return;
  __shared__ float4 ys[kTile];
  const float s = st->sx;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * (128 * RPT) + threadIdx.x;
  float4 xv[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int64_t row = row0 + r * 128;
    xv[r] = row < m ? scale_pt(xt4[row], s) : make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
  }
  const int64_t n_begin = static_cast<int64_t>(blockIdx.y) * n_per_split;
  const int64_t n_end = min(n, n_begin + n_per_split);
  double d0[RPT], dx[RPT], dy[RPT], dz[RPT], dv[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) d0[r] = dx[r] = dy[r] = dz[r] = dv[r] = 0.0;

  for (int64_t base = n_begin; base < n_end; base += kTile) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), n_end - base));
    __syncthreads();
    for (int i = threadIdx.x; i < kTile; i += 128) {
      // padding column: far away and b = -inf → weight exactly 0
      ys[i] = i < cnt ? scale_pt(y4b[base + i], s)
                      : make_float4(kPadCoord, kPadCoord, kPadCoord, -INFINITY);
    }
    __syncthreads();
    float f0[RPT], fx[RPT], fy[RPT], fz[RPT], fv[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) f0[r] = fx[r] = fy[r] = fz[r] = fv[r] = 0.f;
    const int cnt8 = (cnt + 7) & ~7;
    for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 yv = ys[j + u];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const float t = sqdist(yv, xv[r]);
          const float w = ex2_approx(yv.w - t);
          f0[r] += w;
          fx[r] = __fmaf_rn(w, yv.x, fx[r]);
          fy[r] = __fmaf_rn(w, yv.y, fy[r]);
          fz[r] = __fmaf_rn(w, yv.z, fz[r]);
          fv[r] = __fmaf_rn(w, t, fv[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      d0[r] += f0[r];
      dx[r] += fx[r];
      dy[r] += fy[r];
      dz[r] += fz[r];
      dv[r] += fv[r];
    }
  }
  const int64_t sp = static_cast<int64_t>(blockIdx.y) * 5 * m;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int64_t row = row0 + r * 128;
    if (row < m) {
      part[sp + 0 * m + row] = d0[r];
      part[sp + 1 * m + row] = dx[r];
      part[sp + 2 * m + row] = dy[r];
      part[sp + 3 * m + row] = dz[r];
      part[sp + 4 * m + row] = dv[r];
    }
  }
}

// Row finalisation shared by the combine and the fallback.
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

__global__ void estep_row_combine_kernel(const double* __restrict__ part, int splits, int64_t m,
                                         int64_t n, const double* __restrict__ xt64,
                                         RowOut out, YStats ys, int32_t* __restrict__ flag_list,
                                         int32_t* __restrict__ flag_count, IterState* st) {
  if (!st->active) return;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= m) return;
  double a0 = 0, ax = 0, ay = 0, az = 0, av = 0;
  for (int sp = 0; sp < splits; ++sp) {
    const double* p = part + static_cast<int64_t>(sp) * 5 * m;
    a0 += p[row];
    ax += p[m + row];
    ay += p[2 * m + row];
    az += p[3 * m + row];
    av += p[4 * m + row];
  }
  if (!(a0 >= static_cast<double>(n) * 0x1p-76)) {
    const int slot = atomicAdd(flag_count, 1);
    flag_list[slot] = static_cast<int32_t>(row);
    return;
  }
  finalize_row(row, m, log2(a0), a0, ax, ay, az, av, xt64, derived_scale(st), out, ys, st);
}

// Exact row accumulation for flagged rows (tiny mass): warp per row,
// max-shifted, fp64 accumulation.
__global__ void estep_row_fallback_kernel(const float4* __restrict__ xt4, int64_t m,
                                          const float4* __restrict__ y4b, int64_t n,
                                          const double* __restrict__ xt64, RowOut out, YStats ys,
                                          const int32_t* __restrict__ flag_list,
                                          const int32_t* __restrict__ flag_count,
                                          IterState* st) {
  if (!st->active) return;
  const int count = *flag_count;
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  const float s = st->sx;
  for (int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count; w += warps) {
    const int64_t row = flag_list[w];
    const float4 xv = scale_pt(xt4[row], s);
    float lmax = -INFINITY;
    for (int64_t j = lane; j < n; j += 32) {
      const float4 yv = scale_pt(y4b[j], s);
      lmax = fmaxf(lmax, yv.w - sqdist(yv, xv));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    double a0 = 0, ax = 0, ay = 0, az = 0, av = 0;
    if (lmax > -INFINITY) {
      for (int64_t j = lane; j < n; j += 32) {
        const float4 yv = scale_pt(y4b[j], s);
        const float t = sqdist(yv, xv);
        const double wgt = exp2(static_cast<double>(yv.w - t) - static_cast<double>(lmax));
        a0 += wgt;
        ax += wgt * yv.x;
        ay += wgt * yv.y;
        az += wgt * yv.z;
        av += wgt * t;
      }
    }
    a0 = warp_sum(a0);
    ax = warp_sum(ax);
    ay = warp_sum(ay);
    az = warp_sum(az);
    av = warp_sum(av);
    if (lane == 0) {
      const double log2p1 = a0 > 0 ? static_cast<double>(lmax) + log2(a0) : -INFINITY;
      finalize_row(row, m, log2p1, a0, ax, ay, az, av, xt64, derived_scale(st), out, ys, st);
    }
  }
}

// ---------------------------------------------------------------------------
// Host-side launcher.

EStepPlan make_estep_plan(int64_t m, int64_t n, int sm_count) {
  EStepPlan p;
  const int target = sm_count * 8;
  p.col_blocks = ceil_div(n, 128 * kColsPerThread);
  int s1 = ceil_div(target, p.col_blocks);
  s1 = static_cast<int>(std::min<int64_t>(s1, std::max<int64_t>(1, ceil_div(m, 256))));
  p.m_per_split = ceil_div(m, s1);
  p.col_splits = ceil_div(m, p.m_per_split);
  p.row_blocks = ceil_div(m, 128 * kRowsPerThread);
  int s2 = ceil_div(target, p.row_blocks);
  s2 = static_cast<int>(std::min<int64_t>(s2, std::max<int64_t>(1, ceil_div(n, 256))));
  p.n_per_split = ceil_div(n, s2);
  p.row_splits = ceil_div(n, p.n_per_split);
  return p;
}

void launch_estep(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n, int d,
                  double omega, IterState* st, uint64_t* stamps, cudaStream_t stream,
                  cudaEvent_t mid) {
  estep_prologue_kernel<<<1, 1, 0, stream>>>(st, m, n, d, omega, b.flags_count, stamps);
  FCPD_LAUNCH_CHECK();
  estep_col_kernel<kColsPerThread>
      <<<dim3(p.col_blocks, p.col_splits), 128, 0, stream>>>(b.xt4, m, b.y4b, n, p.m_per_split,
                                                             st, b.col_part);
  FCPD_LAUNCH_CHECK();
  estep_col_combine_kernel<<<ceil_div(n, 256), 256, 0, stream>>>(
      b.col_part, p.col_splits, m, n, b.y4b, b.b2, b.pt1, b.col_flags, b.flags_count, st);
  FCPD_LAUNCH_CHECK();
  estep_col_fallback_kernel<<<148, 256, 0, stream>>>(b.xt4, m, b.y4b, b.b2, b.pt1, b.col_flags,
                                                     b.flags_count, st);
  FCPD_LAUNCH_CHECK();
  if (mid) FCPD_CUDA(cudaEventRecord(mid, stream));
  estep_row_kernel<kRowsPerThread>
      <<<dim3(p.row_blocks, p.row_splits), 128, 0, stream>>>(b.xt4, m, b.y4b, n, p.n_per_split,
                                                             st, b.row_part);
  FCPD_LAUNCH_CHECK();
  estep_row_combine_kernel<<<ceil_div(m, 256), 256, 0, stream>>>(
      b.row_part, p.row_splits, m, n, b.xt64, b.out, b.ystats, b.row_flags, b.flags_count + 1,
      st);
  FCPD_LAUNCH_CHECK();
  estep_row_fallback_kernel<<<148, 256, 0, stream>>>(b.xt4, m, b.y4b, n, b.xt64, b.out,
                                                     b.ystats, b.row_flags, b.flags_count + 1,
                                                     st);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
