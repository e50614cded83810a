// mstep.cuh — M-step / transform / σ² launch interface (see mstep.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "estep.cuh"

namespace fcpd {

constexpr int kColsumThreads = 256;
constexpr int kColsPerBlock = 4 * kColsumThreads;  // 1024 columns per column block

// Stream-K plan for "column sums of a row-major matrix weighted by a per-row
// 3-vector": the rows × column-blocks work units (one 4 KB row segment each)
// are split evenly over `grid` persistent CTAs; CTA g writes one fp64
// partial per column block it touches (slot k < kmax).
struct ColsumPlan {
  int64_t rows = 0, cols = 0, cols4 = 0;
  int col_blocks = 0;
  int64_t units = 0;
  int grid = 0;
  int kmax = 0;
  bool bulk = true;  // cp.async.bulk ring (default) or register-staged LDG
  // spectral truncation (IterState::keff): 0 none, 1 the first keff columns
  // (z = Qᵀ R over Q), 2 the first keff rows (V = Q g over Qᵀ)
  int trunc = 0;
  size_t part_doubles() const {
    return static_cast<size_t>(grid) * kmax * 3 * kColsPerBlock;
  }
};

// Row dot products z = Qᵀ·R over the contiguous (truncated) prefix of Qᵀ's
// rows (mstep.cu rowdot_bulk_kernel): units of 8 rows × 1024 columns.
struct RdGeom {
  int64_t rows = 0, cols = 0, lda = 0;  // eigenvector rows, model columns, row stride
  int64_t col_blocks = 0, units = 0;
  int grid = 0, kmax = 0;
  int trunc = 0;  // rows stop at IterState::keff
};
struct RowdotPlan {
  RdGeom g;
  size_t part_doubles() const;
};
RowdotPlan make_rowdot_plan(int64_t k, int64_t m, int64_t lda, int sm_count);
void launch_rowdot(const RowdotPlan& p, const float* qt, const float4* v, double* part,
                   const IterState* st, uint64_t* stamps, int stamp_slot, cudaStream_t stream);
// z = Σ slots per eigenvector; with lam: c = z/(λ + λ_reg σ²), g = λnum·c;
// with z_out (distributed): z itself, SoA 3×K, zeros past the streamed rows.
void launch_rowdot_reduce(const RowdotPlan& p, const double* part, int64_t k, const double* lam,
                          const double* lam_num, double lambda_reg, double* coef, float4* g4,
                          double* z_out, IterState* st, cudaStream_t stream);

// ctas_per_sm: resident bulk CTAs per SM the grid assumes (2 = whole GPU).
ColsumPlan make_colsum_plan(int64_t rows, int64_t cols, int sm_count, int ctas_per_sm = 2);

// The last step of an iteration (one thread): σ² = tot/(D·M) with the
// reference's checks (solvers.hpp:173-175), the clamp count
// (registration.hpp:153), the trace, the next E-step's scalars, and the early
// stop (:159-161).  Shared by sigma_final_kernel, the fused M-step's last CTA
// and the distributed sigma_final_gathered_kernel.
__device__ __forceinline__ void finish_iteration_sigma(IterState* st, double tot, int64_t m, int d,
                                                       int early_stop, double* trace,
                                                       uint64_t* stamps) {
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
  estep_scalars_for_next(st, next, it + 1);  // the next E-step's σ², scale, log c
  if (stamps) stamps[4 * it + 3] = globaltimer();
  if (early_stop && delta < 1e-10) st->active = 0;
}

// Effective spectral rank by a parallel two-round search, for a whole CTA
// (every thread gets the result; all threads must call).  The filter
// f_k = λnum_k/(λ_k + λ_reg σ²) is non-increasing along the descending
// spectrum, so the kept eigenpairs are the prefix before the first f_k < tau:
// round 1 samples blockDim.x evenly spaced k, round 2 scans the bracket that
// holds the first failing sample — two dependent loads instead of log2 K.
__device__ __forceinline__ int64_t cta_spectral_rank(const double* lam, const double* lam_num,
                                                     int64_t k, double c, double tau) {
  __shared__ int first_t;
  __shared__ long long first_i;
  const int t = threadIdx.x, T = blockDim.x;
  auto fails = [&](int64_t i) {
    const double diag = lam[i] + c;
    const double f = diag > 0.0 ? lam_num[i] / diag : 1.0;
    return !(f >= tau);
  };
  auto sample = [&](int64_t j) { return j * k / T; };  // i_0 = 0 < i_1 < … (k ≥ T) or repeats
  if (t == 0) first_t = T;
  __syncthreads();
  if (sample(t) < k && fails(sample(t))) atomicMin(&first_t, t);
  __syncthreads();
  // failing indices form a suffix [first, k): first ∈ (i_{t*−1}, i_{t*}]
  const int ts = first_t;
  const int64_t lo = ts > 0 ? sample(ts - 1) + 1 : 0;
  const int64_t hi = ts < T ? sample(ts) : k;
  if (t == 0) first_i = hi;
  __syncthreads();
  for (int64_t i = lo + t; i < hi; i += T)
    if (fails(i)) atomicMin(&first_i, static_cast<long long>(i));
  __syncthreads();
  const int64_t keep = first_i;
  __syncthreads();  // first_* may be reused by a later call
  return keep;
}

// Effective spectral rank of this iteration → st->keff (multiple of 4):
// the leading eigenpairs whose filter λnum_k/(λ_k + λ_reg σ²) ≥ tau (the
// filter decreases along the descending spectrum); tau ≤ 0 → all K.
void launch_spectral_rank(const double* lam, const double* lam_num, int64_t k, double lambda_reg,
                          double tau, IterState* st, cudaStream_t stream);
// coef = z / (λ + λ_reg σ²_m) from full-K partials (final coefficients when
// the iterations streamed a truncated basis)
void launch_zcoef(const ColsumPlan& p, const double* part, const double* lam, double lambda_reg,
                  double* coef, const IterState* st, cudaStream_t stream);

// distributed final coefficients: coef = z / (λ + λ_reg σ²_m), z all-reduced
void launch_zcoef_full(const double* z, int64_t k, const double* lam, double lambda_reg,
                       double* coef, const IterState* st, cudaStream_t stream);

// part ← partials of Σ_r A[r][c]·v[r].d (d < 3); A row-major fp32, lda % 4 == 0.
void launch_colsum(const ColsumPlan& p, const float* A, int64_t lda, const float4* v,
                   double* part, const IterState* st, uint64_t* stamps, int stamp_slot,
                   cudaStream_t stream);

// z = Σ partials (column c ↔ basis index k); c = z/(λ + λ_reg σ²); g = λnum·c.
void launch_zreduce(const ColsumPlan& p, const double* part, const double* lam,
                    const double* lam_num, double lambda_reg, double* coef, float4* g4,
                    IterState* st, cudaStream_t stream);

// x̃new = X + Σ partials (column c ↔ model point m); per-row σ² terms; σ².
void launch_transform_sigma(const ColsumPlan& p, const double* part, const double* x0,
                            double* xt64, double* xt_prev, float4* xt4,
                            const double* ptilde_y, const double* var, double* sig_part,
                            int d, int early_stop, double* trace, IterState* st,
                            uint64_t* stamps, cudaStream_t stream);

// Number of blocks (= σ² partials) launch_transform_* uses for m rows.
int transform_sigma_blocks(int64_t m);

// Pieces for the distributed path.
int launch_transform_rows(const ColsumPlan& p, const double* part, int64_t m_valid,
                          const double* x0, double* xt64, double* xt_prev, float4* xt4,
                          const double* ptilde_y, const double* var, double* sig_part,
                          IterState* st, uint64_t* stamps, cudaStream_t stream);
void launch_sigma_final(const double* sig_part, int blocks, int64_t m_global, int d,
                        int early_stop, double* trace, IterState* st, uint64_t* stamps,
                        cudaStream_t stream);
void launch_zsum(const ColsumPlan& p, const double* part, double* z, const IterState* st,
                 cudaStream_t stream);
void launch_zfilter(const double* z, int64_t k, const double* lam, const double* lam_num,
                    double lambda_reg, double* coef, float4* g4, IterState* st,
                    cudaStream_t stream);

// The whole M-step (z, solve/filter, V, transform, σ²) as one cooperative
// kernel (mstep_fused.cu): single GPU, for streamed bases that stay in L2.
struct MstepFusedArgs {
  const float* q;   // Q row-major, M × kpad fp32
  int64_t kpad, k;  // row stride, eigenpairs
  const double* lam;
  const double* lam_num;
  double lambda_reg, tau;
  int trunc;  // spectral truncation on (keff from tau)
  const float4* resid4;  // R = P̃Y − X
  double* zpart;         // [k][grid][3]
  double* coef;          // 3 × k SoA
  float4* g4;            // kpad (the padding columns of the last quad get g = 0)
  const double* x0;
  double* xt64;
  double* xt_prev;
  float4* xt4;
  const double* ptilde_y;
  const double* var;
  double* sig_part;  // [grid]
  int32_t* done;     // last-CTA counter (zero before the first launch; self-resetting)
  int64_t m;
  int d, early_stop;
  double* trace;
  IterState* st;
  uint64_t* stamps;
};
int mstep_fused_grid(int sm_count);
void launch_mstep_fused(const MstepFusedArgs& args, int grid, cudaStream_t stream);

// One-kernel EM iteration for small problems (mstep_fused.cu
// small_iter_kernel): both E-step passes with CTA-owned columns / rows, then
// the fused M-step, in one cooperative launch on the fused M-step's grid.
struct SmallIterArgs {
  MstepFusedArgs ms;  // the M-step (and st, xt4, xt64, m)
  float4* y4b;        // scene (x, y, z, b_n): .w written by pass 1
  double* b2;         // b_n fp64
  int64_t n;
  RowOut out;         // P̃Y, var, log2 P1, degenerate, R = P̃Y − X
  YStats ys;
  unsigned long long* counters;  // session counters (pairs by form)
};
bool small_iter_fits(int64_t m, int64_t n);
void launch_small_iter(const SmallIterArgs& args, int grid, cudaStream_t stream);

// out = (x0 or 0) + Σ partials, D columns.
void launch_vreduce_add(const ColsumPlan& p, const double* part, const double* x0, int d,
                        double* out, cudaStream_t stream);

}  // namespace fcpd
