// mstep.cu — Fast-CPD M-step, transform and σ² update for sm_100a.
//
// The reference (solvers.hpp:61-73, :138-155, :160-176; registration.hpp:136)
// computes per iteration
//     R = P̃Y − X,  z = Uᵀ R,  W = U diag(1/(λ_i + λσ²)) z,
//     x̃ = X + Φ W  (full rank)  or  X + U Λ Uᵀ W  (low rank),
//     σ² = (tr(Yᵀ d(P̃ᵀ1) Y) − 2 tr(P̃Yᵀ x̃) + tr(x̃ᵀ x̃)) / (D M).
// Algebraically ΦW = U diag(λ_raw/(λ+λσ²)) z (full rank: Φ = U Λ_raw Uᵀ) and
// U Λ Uᵀ W = U diag(λ/(λ+λσ²)) z (low rank), so one iteration is exactly two
// streaming passes over the basis:
//     z = Qᵀ R        (colsum over Q,  M×K row-major fp32)
//     V = Q (f ⊙ z)   (colsum over Qᵀ, K×M row-major fp32)
// Both are "column sums of a row-major matrix weighted by a per-row 3-vector"
// — the same kernel.  Storing Q and Qᵀ (2× the basis, ≤ 3.2 GB at M=20k)
// makes both passes fully coalesced single reads of HBM.  fp32 products,
// fp32 accumulation over 16-row groups, fp64 accumulation above that, and a
// fixed-order fp64 reduction across row blocks (bitwise reproducible).
//
// σ² uses the cancellation-free per-row form: with
// Δ̄_m = (P̃Y)_m − x̃old_m, V_m = Σ_n P̃_mn‖y_n − x̃old_m‖², δ = x̃new − x̃old,
//     σ² = Σ_m [V_m − 2 δ_m·Δ̄_m + ‖δ_m‖²] / (D M),
// algebraically identical to the reference trace form because rows of P̃
// sum to one.

#include <cuda_runtime.h>

#include "common.cuh"
#include "mstep.cuh"

namespace fcpd {

namespace {
constexpr int kColsumThreads = 256;
constexpr int kRowGroup = 16;  // rows per fp32 sub-accumulation
}  // namespace

// partial[rb][d][c] = Σ_{r in block rb} A[r][c] · v[r].d   (d < 3)
__global__ void __launch_bounds__(kColsumThreads)
    colsum_kernel(const float* __restrict__ A, int64_t lda, int64_t rows, int64_t cols4,
                  const float4* __restrict__ v, int64_t rows_per_block,
                  double* __restrict__ part, int64_t part_ld, const IterState* __restrict__ st,
                  uint64_t* stamps, int stamp_slot) {
  if (st && !st->active) return;
  if (stamps && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    stamps[4 * st->iter + stamp_slot] = globaltimer();
  extern __shared__ float4 vs[];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  const int nr = static_cast<int>(r1 - r0);
  for (int i = threadIdx.x; i < nr; i += kColsumThreads) vs[i] = v[r0 + i];
  __syncthreads();
  const int64_t c4 = static_cast<int64_t>(blockIdx.x) * kColsumThreads + threadIdx.x;
  if (c4 >= cols4) return;
  const float4* a = reinterpret_cast<const float4*>(A + r0 * lda) + c4;
  const int64_t ld4 = lda >> 2;
  double acc[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;

  int r = 0;
  for (; r + kRowGroup <= nr; r += kRowGroup) {
    float4 q[kRowGroup];
#pragma unroll
    for (int u = 0; u < kRowGroup; ++u) q[u] = __ldcs(a + static_cast<int64_t>(r + u) * ld4);
    float f[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i][0] = f[i][1] = f[i][2] = 0.f;
#pragma unroll
    for (int u = 0; u < kRowGroup; ++u) {
      const float4 w = vs[r + u];
      const float qq[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        f[i][0] = __fmaf_rn(qq[i], w.x, f[i][0]);
        f[i][1] = __fmaf_rn(qq[i], w.y, f[i][1]);
        f[i][2] = __fmaf_rn(qq[i], w.z, f[i][2]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i][0] += f[i][0];
      acc[i][1] += f[i][1];
      acc[i][2] += f[i][2];
    }
  }
  for (; r < nr; ++r) {
    const float4 q = __ldcs(a + static_cast<int64_t>(r) * ld4);
    const float4 w = vs[r];
    const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i][0] += static_cast<double>(qq[i] * w.x);
      acc[i][1] += static_cast<double>(qq[i] * w.y);
      acc[i][2] += static_cast<double>(qq[i] * w.z);
    }
  }
  double* out = part + static_cast<int64_t>(blockIdx.y) * 3 * part_ld + 4 * c4;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double2* o = reinterpret_cast<double2*>(out + d * part_ld);
    o[0] = make_double2(acc[0][d], acc[1][d]);
    o[1] = make_double2(acc[2][d], acc[3][d]);
  }
}

// z_k = Σ_rb partial; solve + filter (solvers.hpp:66-72):
//   c_k = z_k / (λ_k + λ_reg σ²)   (W = Q c, kept for `coefficients`)
//   g_k = λnum_k · c_k             (ΦW = Q g)
__global__ void zreduce_filter_kernel(const double* __restrict__ part, int blocks, int64_t k,
                                      int64_t part_ld, const double* __restrict__ lam,
                                      const double* __restrict__ lam_num, double lambda_reg,
                                      double* __restrict__ coef, float4* __restrict__ g4,
                                      IterState* st) {
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double z0 = 0, z1 = 0, z2 = 0;
  for (int b = 0; b < blocks; ++b) {
    const double* p = part + static_cast<int64_t>(b) * 3 * part_ld;
    z0 += p[i];
    z1 += p[part_ld + i];
    z2 += p[2 * part_ld + i];
  }
  // σ² of this iteration's E-step, unclamped (registration.hpp:137)
  const double diag = lam[i] + lambda_reg * st->sigma2;
  if (!(diag > 0.0)) set_error(st, kDevSolveDiag, diag);
  const double inv = 1.0 / diag;
  coef[i] = z0 * inv;
  coef[k + i] = z1 * inv;
  coef[2 * k + i] = z2 * inv;
  const double f = lam_num[i] * inv;
  g4[i] = make_float4(static_cast<float>(z0 * f), static_cast<float>(z1 * f),
                      static_cast<float>(z2 * f), 0.f);
}

// x̃new = X + V; per-row σ² terms; block partial sums (fixed order).
__global__ void __launch_bounds__(256)
    transform_sigma_kernel(const double* __restrict__ part, int blocks, int64_t m,
                           int64_t part_ld, const double* __restrict__ x0, double* xt64,
                           double* __restrict__ xt_prev, float4* __restrict__ xt4,
                           const double* __restrict__ ptilde_y, const double* __restrict__ var,
                           double* __restrict__ sig_part, IterState* st, uint64_t* stamps) {
  if (!st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0) stamps[4 * st->iter + 2] = globaltimer();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (i < m) {
    double v0 = 0, v1 = 0, v2 = 0;
    for (int b = 0; b < blocks; ++b) {
      const double* p = part + static_cast<int64_t>(b) * 3 * part_ld;
      v0 += p[i];
      v1 += p[part_ld + i];
      v2 += p[2 * part_ld + i];
    }
    const double o0 = xt64[i], o1 = xt64[m + i], o2 = xt64[2 * m + i];
    const double n0 = x0[i] + v0, n1 = x0[m + i] + v1, n2 = x0[2 * m + i] + v2;
    const double d0 = n0 - o0, d1 = n1 - o1, d2 = n2 - o2;
    const double a0 = ptilde_y[i] - o0, a1 = ptilde_y[m + i] - o1, a2 = ptilde_y[2 * m + i] - o2;
    term = var[i] - 2.0 * (d0 * a0 + d1 * a1 + d2 * a2) + (d0 * d0 + d1 * d1 + d2 * d2);
    if (xt_prev) {
      xt_prev[i] = o0;
      xt_prev[m + i] = o1;
      xt_prev[2 * m + i] = o2;
    }
    xt64[i] = n0;
    xt64[m + i] = n1;
    xt64[2 * m + i] = n2;
    xt4[i] = make_float4(static_cast<float>(n0), static_cast<float>(n1),
                         static_cast<float>(n2), 0.f);
  }
  // deterministic block reduction
  __shared__ double red[8];
  term = warp_sum(term);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = term;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) s += red[w];
    sig_part[blockIdx.x] = s;
  }
}

// σ² = Σ partials / (D·M); reference checks (solvers.hpp:173-175),
// clamp count (registration.hpp:153), trace, early stop (:159-161).
__global__ void sigma_final_kernel(const double* __restrict__ sig_part, int blocks, int64_t m,
                                   int d, int early_stop, double* __restrict__ trace,
                                   IterState* st, uint64_t* stamps) {
  if (!st->active) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < blocks; b += blockDim.x) s += sig_part[b];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double tot = 0.0;
  for (int w = 0; w < (blockDim.x >> 5); ++w) tot += red[w];
  const double val = tot / (static_cast<double>(d) * static_cast<double>(m));
  if (val < -1e-8) set_error(st, kDevNegVariance, val);
  const double next = fmax(val, kSigma2Floor);
  if (next <= kSigma2Floor) st->sigma2_clamps += 1;
  const int it = st->iter;
  trace[it] = next;
  const double delta = fabs(next - st->sigma2);
  st->sigma2 = next;
  st->iters_run = it + 1;
  st->iter = it + 1;
  if (stamps) stamps[4 * it + 3] = globaltimer();
  if (early_stop && delta < 1e-10) st->active = 0;
}

// ---------------------------------------------------------------------------

ColsumPlan make_colsum_plan(int64_t rows, int64_t cols, int sm_count) {
  ColsumPlan p;
  p.cols4 = (cols + 3) / 4;
  p.col_blocks = ceil_div(p.cols4, kColsumThreads);
  // aim for ~4 resident waves; at least 64 rows per block, at most 2048
  const int64_t target = static_cast<int64_t>(sm_count) * 8;
  int64_t row_blocks = std::max<int64_t>(1, target / p.col_blocks);
  int64_t rpb = (rows + row_blocks - 1) / row_blocks;
  rpb = std::max<int64_t>(64, std::min<int64_t>(2048, rpb));
  rpb = (rpb + kRowGroup - 1) / kRowGroup * kRowGroup;
  p.rows_per_block = rpb;
  p.row_blocks = ceil_div(rows, rpb);
  return p;
}

void launch_colsum(const ColsumPlan& p, const float* A, int64_t lda, int64_t rows,
                   const float4* v, double* part, int64_t part_ld, const IterState* st,
                   uint64_t* stamps, int stamp_slot, cudaStream_t stream) {
  const size_t smem = sizeof(float4) * p.rows_per_block;
  colsum_kernel<<<dim3(p.col_blocks, p.row_blocks), kColsumThreads, smem, stream>>>(
      A, lda, rows, p.cols4, v, p.rows_per_block, part, part_ld, st, stamps, stamp_slot);
  FCPD_LAUNCH_CHECK();
}

void launch_zreduce(const double* part, int blocks, int64_t k, int64_t part_ld,
                    const double* lam, const double* lam_num, double lambda_reg, double* coef,
                    float4* g4, IterState* st, cudaStream_t stream) {
  zreduce_filter_kernel<<<ceil_div(k, 256), 256, 0, stream>>>(part, blocks, k, part_ld, lam,
                                                              lam_num, lambda_reg, coef, g4, st);
  FCPD_LAUNCH_CHECK();
}

void launch_transform_sigma(const double* part, int blocks, int64_t m, int64_t part_ld,
                            const double* x0, double* xt64, double* xt_prev, float4* xt4,
                            const double* ptilde_y, const double* var, double* sig_part,
                            int d, int early_stop, double* trace, IterState* st,
                            uint64_t* stamps, cudaStream_t stream) {
  const int nb = ceil_div(m, 256);
  transform_sigma_kernel<<<nb, 256, 0, stream>>>(part, blocks, m, part_ld, x0, xt64, xt_prev,
                                                 xt4, ptilde_y, var, sig_part, st, stamps);
  FCPD_LAUNCH_CHECK();
  sigma_final_kernel<<<1, 256, 0, stream>>>(sig_part, nb, m, d, early_stop, trace, st, stamps);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd

namespace fcpd {

// out = X + Σ_b part[b]  (apply_transform_lowrank epilogue, no σ² terms)
__global__ void vreduce_add_kernel(const double* __restrict__ part, int blocks, int64_t m,
                                   int64_t part_ld, const double* __restrict__ x0, int d,
                                   double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int c = 0; c < d; ++c) {
    double v = 0.0;
    for (int b = 0; b < blocks; ++b) v += part[(static_cast<int64_t>(b) * 3 + c) * part_ld + i];
    out[c * m + i] = x0[c * m + i] + v;
  }
}

void launch_vreduce_add(const double* part, int blocks, int64_t m, int64_t part_ld,
                        const double* x0, int d, double* out, cudaStream_t stream) {
  vreduce_add_kernel<<<ceil_div(m, 256), 256, 0, stream>>>(part, blocks, m, part_ld, x0, d, out);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
