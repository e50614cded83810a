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
constexpr int kCombineLanes = 8; // lanes cooperating on one row/column reduction
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

__device__ __forceinline__ float4 box_min(float4 a, float4 b) {
  return make_float4(fminf(a.x, b.x), fminf(a.y, b.y), fminf(a.z, b.z), 0.f);
}
__device__ __forceinline__ float4 box_max(float4 a, float4 b) {
  return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), 0.f);
}
// smallest squared distance between two boxes (0 if they overlap)
__device__ __forceinline__ float box_mindist2(float4 alo, float4 ahi, float4 blo, float4 bhi) {
  const float dx = fmaxf(0.f, fmaxf(alo.x - bhi.x, blo.x - ahi.x));
  const float dy = fmaxf(0.f, fmaxf(alo.y - bhi.y, blo.y - ahi.y));
  const float dz = fmaxf(0.f, fmaxf(alo.z - bhi.z, blo.z - ahi.z));
  // shrink by one part in 2^20: fp32 rounding of the bound never culls a pair
  // the exact geometry would keep
  return (dx * dx + dy * dy + dz * dz) * (1.f - 0x1p-20f);
}
// largest squared distance between points of two boxes
__device__ __forceinline__ float box_maxdist2(float4 alo, float4 ahi, float4 blo, float4 bhi) {
  const float dx = fmaxf(ahi.x - blo.x, bhi.x - alo.x);
  const float dy = fmaxf(ahi.y - blo.y, bhi.y - alo.y);
  const float dz = fmaxf(ahi.z - blo.z, bhi.z - alo.z);
  return (dx * dx + dy * dy + dz * dz) * (1.f + 0x1p-20f);
}

}  // namespace

// ---------------------------------------------------------------------------
// Iteration prologue: σ² floor + clamp count (correspondence.hpp:43-47,
// registration.hpp:122), coordinate scale, outlier constant (:61-66).
__global__ void estep_prologue_kernel(IterState* st, int64_t m, int64_t n, int d,
                                      double omega, int32_t* flags_count, uint64_t* stamps) {
  if (!st->active) return;
  if (stamps) stamps[4 * st->iter + 0] = globaltimer();
  for (int i = 0; i <= kMaxRowChunks; ++i) flags_count[i] = 0;  // column + per-chunk row lists
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
//
// f32x2 packing (FADD2/FMUL2/FFMA2, sm_100): each thread owns CP column
// pairs; every packed op evaluates two (m, n) pairs in one issue slot, so
// per pair the pass costs 3.5 issue slots of FP32 work + 1 MUFU.EX2 and is
// bound by the 16 ex2/clk/SM SFU rate.  Each lane of a packed op rounds
// exactly like the scalar op, so t_mn is bitwise identical to sqdist() used
// by pass 2 and the fallbacks.  Shared memory holds each model point as
// (−x,−x,−y,−y),(−z,−z) so a broadcast LDS yields the packed operand.
template <int CP>
__global__ void __launch_bounds__(128)
    estep_col_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4,
                     int64_t n, int64_t m_per_split, const IterState* __restrict__ st,
                     double* __restrict__ part, CullInfo cull) {
  if (!st->active) return;
  __shared__ float4 xa[kTile];  // (−x, −x, −y, −y)
  __shared__ float2 xb[kTile];  // (−z, −z)
  const float s = st->sx;
  const float s2 = s * s;
  // tile culling: this CTA's 256 columns vs each 256-point model tile
  float4 blo = make_float4(0.f, 0.f, 0.f, 0.f), bhi = blo;
  float cut = INFINITY;
  if (cull.enabled) {  // a column block is exactly one 256-point scene tile
    blo = cull.ylo[blockIdx.x];
    bhi = cull.yhi[blockIdx.x];
    cut = s2 * cull.col_bound[blockIdx.x] + cull.margin1;
  }
  int evaluated = 0;
  // column pair p of this thread: cols c, c+1 with c = base + p·256 + 2·tid
  const int64_t cbase = static_cast<int64_t>(blockIdx.x) * (256 * CP) + 2 * threadIdx.x;
  float2 yx[CP], yy[CP], yz[CP];
#pragma unroll
  for (int p = 0; p < CP; ++p) {
    const int64_t c = cbase + p * 256;
    const float4 a = c < n ? scale_pt(y4[c], s) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b = c + 1 < n ? scale_pt(y4[c + 1], s) : make_float4(0.f, 0.f, 0.f, 0.f);
    yx[p] = make_float2(a.x, b.x);
    yy[p] = make_float2(a.y, b.y);
    yz[p] = make_float2(a.z, b.z);
  }
  const int64_t m_begin = static_cast<int64_t>(blockIdx.y) * m_per_split;
  const int64_t m_end = min(m, m_begin + m_per_split);
  double dsum[CP][2];
#pragma unroll
  for (int p = 0; p < CP; ++p) dsum[p][0] = dsum[p][1] = 0.0;

  for (int64_t base = m_begin; base < m_end; base += kTile) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), m_end - base));
    if (cull.enabled) {  // uniform across the CTA (same data, same math)
      const int64_t tj = base / kTile;  // m_per_split is a multiple of kTile
      if (s2 * box_mindist2(blo, bhi, cull.xlo[tj], cull.xhi[tj]) > cut) continue;
    }
    ++evaluated;
    __syncthreads();
    for (int i = threadIdx.x; i < kTile; i += 128) {
      const float4 v = i < cnt ? scale_pt(xt4[base + i], s)
                               : make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
      xa[i] = make_float4(-v.x, -v.x, -v.y, -v.y);
      xb[i] = make_float2(-v.z, -v.z);
    }
    __syncthreads();
    float2 fsum[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) fsum[p] = make_float2(0.f, 0.f);
    const int cnt8 = (cnt + 7) & ~7;
    for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 a = xa[j + u];
        const float2 nx = make_float2(a.x, a.y), ny = make_float2(a.z, a.w);
        const float2 nz = xb[j + u];
#pragma unroll
        for (int p = 0; p < CP; ++p) {
          const float2 dx = __fadd2_rn(yx[p], nx);
          const float2 dy = __fadd2_rn(yy[p], ny);
          const float2 dz = __fadd2_rn(yz[p], nz);
          float2 t = __fmul2_rn(dx, dx);
          t = __ffma2_rn(dy, dy, t);
          t = __ffma2_rn(dz, dz, t);
          fsum[p] = __fadd2_rn(fsum[p], make_float2(ex2_approx(-t.x), ex2_approx(-t.y)));
        }
      }
    }
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      dsum[p][0] += static_cast<double>(fsum[p].x);
      dsum[p][1] += static_cast<double>(fsum[p].y);
    }
  }
  double* out = part + static_cast<int64_t>(blockIdx.y) * n;
#pragma unroll
  for (int p = 0; p < CP; ++p) {
    const int64_t c = cbase + p * 256;
    if (c < n) out[c] = dsum[p][0];
    if (c + 1 < n) out[c + 1] = dsum[p][1];
  }
  if (cull.counters && threadIdx.x == 0) atomicAdd(cull.counters, (unsigned long long)evaluated);
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
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t col = gid / kCombineLanes;
  const int lane = static_cast<int>(gid % kCombineLanes);
  double sm = 0.0;
  if (col < n)
    for (int s = lane; s < splits; s += kCombineLanes) sm += part[static_cast<int64_t>(s) * n + col];
#pragma unroll
  for (int o = kCombineLanes / 2; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  if (col >= n || lane != 0) return;
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
//
// f32x2 packing over row pairs: per pair 6 packed FP32 issue slots (12
// lane-ops: the FP32 pipe bound) + 1 MUFU.EX2.  Shared memory holds each
// scene point as (y,y,y',y'),(z,z,b,b) so a broadcast LDS yields the packed
// operands; the weight is w = 2^{b − t} (b − t = FFMA2(t, −1, b)).
template <int RP>
__global__ void __launch_bounds__(128)
    estep_row_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4b,
                     int64_t n, int64_t n_per_split, const IterState* __restrict__ st,
                     double* __restrict__ part /* [split][5][m] */, int rb_offset,
                     CullInfo cull) {
  if (!st->active) return;
  __shared__ float4 ya[kTile];  // (yx, yx, yy, yy)
  __shared__ float4 yb[kTile];  // (yz, yz, b, b)
  const float s = st->sx;
  const float s2 = s * s;
  const int64_t rbase =
      static_cast<int64_t>(blockIdx.x + rb_offset) * (256 * RP) + 2 * threadIdx.x;
  // tile culling: this CTA's 256 model rows vs each 256-point scene tile
  float4 blo = make_float4(0.f, 0.f, 0.f, 0.f), bhi = blo;
  float floor_l = -INFINITY;
  if (cull.enabled) {  // a row block is exactly one 256-point model tile
    const int64_t rb = blockIdx.x + rb_offset;
    blo = cull.xlo[rb];
    bhi = cull.xhi[rb];
    floor_l = cull.row_bound[rb] - cull.margin2;
  }
  int evaluated = 0;
  float2 nx[RP], ny[RP], nz[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    const int64_t r = rbase + p * 256;
    const float4 pad = make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
    const float4 a = r < m ? scale_pt(xt4[r], s) : pad;
    const float4 b = r + 1 < m ? scale_pt(xt4[r + 1], s) : pad;
    nx[p] = make_float2(-a.x, -b.x);
    ny[p] = make_float2(-a.y, -b.y);
    nz[p] = make_float2(-a.z, -b.z);
  }
  const int64_t n_begin = static_cast<int64_t>(blockIdx.y) * n_per_split;
  const int64_t n_end = min(n, n_begin + n_per_split);
  // fp64 tile accumulators live in shared memory (thread-private slots,
  // [quantity][row][thread] → conflict-free): keeps registers for the packed
  // pipeline and raises occupancy (the pass is FP32-pipe bound).
  __shared__ double acc_s[5][2 * RP][128];
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int r = 0; r < 2 * RP; ++r) acc_s[k][r][threadIdx.x] = 0.0;
  const float2 minus1 = make_float2(-1.f, -1.f);

  for (int64_t base = n_begin; base < n_end; base += kTile) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), n_end - base));
    if (cull.enabled) {  // L ≤ bmax − s²·mindist² < (row-max lower bound) − margin → skip
      const int64_t tj = base / kTile;  // n_per_split is a multiple of kTile
      const float lub = cull.bminmax[tj].y - s2 * box_mindist2(blo, bhi, cull.ylo[tj], cull.yhi[tj]);
      if (lub < floor_l) continue;
    }
    ++evaluated;
    __syncthreads();
    for (int i = threadIdx.x; i < kTile; i += 128) {
      // padding column: far away and b = −inf → weight exactly 0
      const float4 v = i < cnt ? scale_pt(y4b[base + i], s)
                               : make_float4(kPadCoord, kPadCoord, kPadCoord, -INFINITY);
      ya[i] = make_float4(v.x, v.x, v.y, v.y);
      yb[i] = make_float4(v.z, v.z, v.w, v.w);
    }
    __syncthreads();
    float2 f0[RP], fx[RP], fy[RP], fz[RP], fv[RP];
#pragma unroll
    for (int p = 0; p < RP; ++p)
      f0[p] = fx[p] = fy[p] = fz[p] = fv[p] = make_float2(0.f, 0.f);
    const int cnt8 = (cnt + 7) & ~7;
    for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 a = ya[j + u];
        const float4 c = yb[j + u];
        const float2 Yx = make_float2(a.x, a.y), Yy = make_float2(a.z, a.w);
        const float2 Yz = make_float2(c.x, c.y), B = make_float2(c.z, c.w);
#pragma unroll
        for (int p = 0; p < RP; ++p) {
          const float2 ddx = __fadd2_rn(Yx, nx[p]);
          const float2 ddy = __fadd2_rn(Yy, ny[p]);
          const float2 ddz = __fadd2_rn(Yz, nz[p]);
          float2 t = __fmul2_rn(ddx, ddx);
          t = __ffma2_rn(ddy, ddy, t);
          t = __ffma2_rn(ddz, ddz, t);
          const float2 L = __ffma2_rn(t, minus1, B);
          const float2 w = make_float2(ex2_approx(L.x), ex2_approx(L.y));
          f0[p] = __fadd2_rn(f0[p], w);
          fx[p] = __ffma2_rn(w, Yx, fx[p]);
          fy[p] = __ffma2_rn(w, Yy, fy[p]);
          fz[p] = __ffma2_rn(w, Yz, fz[p]);
          fv[p] = __ffma2_rn(w, t, fv[p]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < RP; ++p) {
      const int t = threadIdx.x;
      acc_s[0][2 * p][t] += f0[p].x;
      acc_s[0][2 * p + 1][t] += f0[p].y;
      acc_s[1][2 * p][t] += fx[p].x;
      acc_s[1][2 * p + 1][t] += fx[p].y;
      acc_s[2][2 * p][t] += fy[p].x;
      acc_s[2][2 * p + 1][t] += fy[p].y;
      acc_s[3][2 * p][t] += fz[p].x;
      acc_s[3][2 * p + 1][t] += fz[p].y;
      acc_s[4][2 * p][t] += fv[p].x;
      acc_s[4][2 * p + 1][t] += fv[p].y;
    }
  }
  const int64_t sp = static_cast<int64_t>(blockIdx.y) * 5 * m;
#pragma unroll
  for (int p = 0; p < RP; ++p)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = rbase + p * 256 + h;
      if (row < m) {
#pragma unroll
        for (int k = 0; k < 5; ++k) part[sp + k * m + row] = acc_s[k][2 * p + h][threadIdx.x];
      }
    }
  if (cull.counters && threadIdx.x == 0)
    atomicAdd(cull.counters + 1, (unsigned long long)evaluated);
}

// ---------------------------------------------------------------------------
// Tile geometry for culling (points are Morton-sorted by the engine, so
// 256-point tiles are spatially compact).

// per-tile axis-aligned box of the first three coordinates (unscaled)
__global__ void tile_bbox_kernel(const float4* __restrict__ p, int64_t count,
                                 float4* __restrict__ lo, float4* __restrict__ hi,
                                 const IterState* __restrict__ st) {
  if (st && !st->active) return;
  __shared__ float red[6][8];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kTile + threadIdx.x;
  float v[6];
  if (i < count) {
    const float4 q = p[i];
    v[0] = v[3] = q.x;
    v[1] = v[4] = q.y;
    v[2] = v[5] = q.z;
  } else {
    v[0] = v[1] = v[2] = INFINITY;
    v[3] = v[4] = v[5] = -INFINITY;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const float w = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = k < 3 ? fminf(v[k], w) : fmaxf(v[k], w);
    }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) red[k][warp] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    float r[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) r[k] = red[k][0];
    for (int w = 1; w < kTile / 32; ++w)
#pragma unroll
      for (int k = 0; k < 6; ++k) r[k] = k < 3 ? fminf(r[k], red[k][w]) : fmaxf(r[k], red[k][w]);
    lo[blockIdx.x] = make_float4(r[0], r[1], r[2], 0.f);
    hi[blockIdx.x] = make_float4(r[3], r[4], r[5], 0.f);
  }
}

// per scene tile: (min b_n, max b_n) after pass 1
__global__ void tile_bminmax_kernel(const float4* __restrict__ y4b, int64_t n,
                                    float2* __restrict__ out, const IterState* __restrict__ st) {
  if (!st->active) return;
  __shared__ float red[2][8];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kTile + threadIdx.x;
  float mn = INFINITY, mx = -INFINITY;
  if (i < n) mn = mx = y4b[i].w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mn;
    red[1][threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kTile / 32; ++w) {
      mn = fminf(red[0][0], red[0][w]);
      mx = fmaxf(red[1][0], red[1][w]);
      red[0][0] = mn;
      red[1][0] = mx;
    }
    out[blockIdx.x] = make_float2(red[0][0], red[1][0]);
  }
}

// pass-1 bound per scene tile: U = min over model tiles of the largest
// possible squared distance → every column has t_min ≤ s²·U.
__global__ void col_bound_kernel(CullInfo cull, float* __restrict__ out, int n_blocks,
                                 const IterState* __restrict__ st) {
  if (!st->active) return;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= n_blocks) return;
  const float4 lo = cull.ylo[b], hi = cull.yhi[b];
  float u = INFINITY;
  for (int j = lane; j < cull.n_xtiles; j += 32)
    u = fminf(u, box_maxdist2(lo, hi, cull.xlo[j], cull.xhi[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u = fminf(u, __shfl_xor_sync(0xffffffffu, u, o));
  if (lane == 0) out[b] = u;
}

// pass-2 bound per model tile: a lower bound on max_n L_mn for every row,
// L_lb = max over scene tiles of (min b − s²·maxdist²).
__global__ void row_bound_kernel(CullInfo cull, float* __restrict__ out, int n_blocks,
                                 const IterState* __restrict__ st) {
  if (!st->active) return;
  const float s2 = st->sx * st->sx;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= n_blocks) return;
  const float4 lo = cull.xlo[b], hi = cull.xhi[b];
  float l = -INFINITY;
  for (int j = lane; j < cull.n_ytiles; j += 32)
    l = fmaxf(l, cull.bminmax[j].x - s2 * box_maxdist2(lo, hi, cull.ylo[j], cull.yhi[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l = fmaxf(l, __shfl_xor_sync(0xffffffffu, l, o));
  if (lane == 0) out[b] = l;
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
                                         int32_t* __restrict__ flag_count, IterState* st,
                                         int64_t r0, int64_t r1) {
  if (!st->active) return;
  // kCombineLanes lanes per row, lane j sums splits j, j+L, … then a fixed
  // xor-tree combines the lanes: deterministic, and L× the memory-level
  // parallelism of one thread per row.  Rows [r0, r1) of this launch.
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = r0 + gid / kCombineLanes;
  const int lane = static_cast<int>(gid % kCombineLanes);
  const bool live = row < r1;
  double a0 = 0, ax = 0, ay = 0, az = 0, av = 0;
  if (live) {
    for (int sp = lane; sp < splits; sp += kCombineLanes) {
      const double* p = part + static_cast<int64_t>(sp) * 5 * m;
      a0 += p[row];
      ax += p[m + row];
      ay += p[2 * m + row];
      az += p[3 * m + row];
      av += p[4 * m + row];
    }
  }
#pragma unroll
  for (int o = kCombineLanes / 2; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    ax += __shfl_xor_sync(0xffffffffu, ax, o);
    ay += __shfl_xor_sync(0xffffffffu, ay, o);
    az += __shfl_xor_sync(0xffffffffu, az, o);
    av += __shfl_xor_sync(0xffffffffu, av, o);
  }
  if (!live || lane != 0) return;
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

// Split the reduction axis so the grid fills whole waves: CTAs are uniform,
// so wave efficiency = T / (ceil(T/slots)·slots) with T = blocks × splits.
// Take the fewest splits reaching ≥ 96 % (or the best found), keeping ≥ 128
// reduction points per split.
static int choose_splits(int blocks, int64_t len, int slots) {
  const int max_s = static_cast<int>(std::max<int64_t>(1, len / 128));
  int best = 1;
  double best_eff = -1.0;
  for (int s = 1; s <= max_s; ++s) {
    const int64_t per = ceil_div(len, s);
    const int real = ceil_div(len, per);  // splits actually produced
    const int64_t t = static_cast<int64_t>(blocks) * real;
    const double waves = std::ceil(static_cast<double>(t) / slots);
    const double eff = static_cast<double>(t) / (waves * slots);
    if (t < slots && s < max_s) continue;  // want at least one full wave
    if (eff >= 0.96) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

EStepPlan make_estep_plan(int64_t m, int64_t n, int sm_count) {
  EStepPlan p;
  int occ_col = 0, occ_row = 0;
  FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ_col, estep_col_kernel<kColsPerThread / 2>, 128, 0));
  FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ_row, estep_row_kernel<kRowsPerThread / 2>, 128, 0));
  p.col_blocks = ceil_div(n, 128 * kColsPerThread);
  const int s1 = choose_splits(p.col_blocks, m, sm_count * std::max(occ_col, 1));
  // splits on 256-point tile boundaries (culling tests whole tiles)
  p.m_per_split = static_cast<int64_t>(ceil_div(ceil_div(m, s1), kTile)) * kTile;
  p.col_splits = ceil_div(m, p.m_per_split);
  p.row_blocks = ceil_div(m, 128 * kRowsPerThread);
  const int s2 = choose_splits(p.row_blocks, n, sm_count * std::max(occ_row, 1));
  p.n_per_split = static_cast<int64_t>(ceil_div(ceil_div(n, s2), kTile)) * kTile;
  p.row_splits = ceil_div(n, p.n_per_split);
  p.chunks = 1;
  return p;
}

void plan_row_chunks(EStepPlan& p, int64_t m, int64_t n, int sm_count, int chunks) {
  int occ_row = 0;
  FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ_row, estep_row_kernel<kRowsPerThread / 2>, 128, 0));
  p.chunks = chunks;
  for (int c = 0; c < chunks; ++c) {
    const int rb = static_cast<int>(static_cast<int64_t>(p.row_blocks) * (c + 1) / chunks -
                                    static_cast<int64_t>(p.row_blocks) * c / chunks);
    const int s = choose_splits(std::max(rb, 1), n, sm_count * std::max(occ_row, 1));
    p.chunk_nps[c] = static_cast<int64_t>(ceil_div(ceil_div(n, s), kTile)) * kTile;
    p.chunk_splits[c] = ceil_div(n, p.chunk_nps[c]);
  }
}

void launch_estep_prologue(IterState* st, int64_t m, int64_t n_global, int d, double omega,
                           int32_t* flags_count, uint64_t* stamps, cudaStream_t stream) {
  estep_prologue_kernel<<<1, 1, 0, stream>>>(st, m, n_global, d, omega, flags_count, stamps);
  FCPD_LAUNCH_CHECK();
}

void launch_tile_bbox(const float4* pts, int64_t count, float4* lo, float4* hi,
                      const IterState* st, cudaStream_t stream) {
  tile_bbox_kernel<<<ceil_div(count, kTile), kTile, 0, stream>>>(pts, count, lo, hi, st);
  FCPD_LAUNCH_CHECK();
}

// Pass 1 (column normalisers) + the culling geometry around it: model-tile
// boxes of this iteration's x̃ and the per-block bounds before, scene-tile
// b ranges and row bounds after (pass 2 reads them).
void launch_estep_pass1(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream) {
  const CullInfo& cu = b.cull;
  if (cu.enabled) {
    launch_tile_bbox(b.xt4, m, b.cullw.xlo, b.cullw.xhi, st, stream);
    col_bound_kernel<<<ceil_div(p.col_blocks, 8), 256, 0, stream>>>(cu, b.cullw.col_bound,
                                                                    p.col_blocks, st);
    FCPD_LAUNCH_CHECK();
  }
  estep_col_kernel<kColsPerThread / 2>
      <<<dim3(p.col_blocks, p.col_splits), 128, 0, stream>>>(b.xt4, m, b.y4b, n, p.m_per_split,
                                                             st, b.col_part, cu);
  FCPD_LAUNCH_CHECK();
  estep_col_combine_kernel<<<ceil_div(n * kCombineLanes, 256), 256, 0, stream>>>(
      b.col_part, p.col_splits, m, n, b.y4b, b.b2, b.pt1, b.col_flags, b.flags_count, st);
  FCPD_LAUNCH_CHECK();
  estep_col_fallback_kernel<<<148, 256, 0, stream>>>(b.xt4, m, b.y4b, b.b2, b.pt1, b.col_flags,
                                                     b.flags_count, st);
  FCPD_LAUNCH_CHECK();
  if (cu.enabled) {
    tile_bminmax_kernel<<<ceil_div(n, kTile), kTile, 0, stream>>>(b.y4b, n, b.cullw.bminmax, st);
    FCPD_LAUNCH_CHECK();
    row_bound_kernel<<<ceil_div(p.row_blocks, 8), 256, 0, stream>>>(cu, b.cullw.row_bound,
                                                                    p.row_blocks, st);
    FCPD_LAUNCH_CHECK();
  }
}

void launch_estep_pass2_partials(const EStepPlan& p, const EStepBuffers& b, int64_t m,
                                 int64_t n, IterState* st, cudaStream_t stream) {
  estep_row_kernel<kRowsPerThread / 2>
      <<<dim3(p.row_blocks, p.row_splits), 128, 0, stream>>>(b.xt4, m, b.y4b, n, p.n_per_split,
                                                             st, b.row_part, 0, b.cull);
  FCPD_LAUNCH_CHECK();
}

void launch_estep(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n, int d,
                  double omega, IterState* st, uint64_t* stamps, cudaStream_t stream,
                  cudaEvent_t mid) {
  estep_prologue_kernel<<<1, 1, 0, stream>>>(st, m, n, d, omega, b.flags_count, stamps);
  FCPD_LAUNCH_CHECK();
  launch_estep_pass1(p, b, m, n, st, stream);
  if (mid) FCPD_CUDA(cudaEventRecord(mid, stream));
  launch_estep_pass2_chunk(p, b, m, n, st, stream, 0, 1);
}

RowChunk row_chunk(const EStepPlan& p, int64_t m, int c, int chunks) {
  RowChunk r;
  r.rb0 = static_cast<int>(static_cast<int64_t>(p.row_blocks) * c / chunks);
  r.rb1 = static_cast<int>(static_cast<int64_t>(p.row_blocks) * (c + 1) / chunks);
  r.r0 = std::min<int64_t>(m, static_cast<int64_t>(r.rb0) * 128 * kRowsPerThread);
  r.r1 = std::min<int64_t>(m, static_cast<int64_t>(r.rb1) * 128 * kRowsPerThread);
  return r;
}

// Pass 2 for the model rows of chunk c of `chunks`: partial sums, combine,
// exact fallback for this chunk's flagged rows (its own list/counter), so
// the rows' P̃Y / residual are final when the launch sequence returns and a
// consumer (the Qᵀ·R stream of the same rows) can start on another stream.
void launch_estep_pass2_chunk(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                              IterState* st, cudaStream_t stream, int c, int chunks) {
  const RowChunk rc = row_chunk(p, m, c, chunks);
  if (rc.rb1 <= rc.rb0) return;
  const bool own = chunks > 1 && p.chunks == chunks;
  const int splits = own ? p.chunk_splits[c] : p.row_splits;
  const int64_t nps = own ? p.chunk_nps[c] : p.n_per_split;
  estep_row_kernel<kRowsPerThread / 2><<<dim3(rc.rb1 - rc.rb0, splits), 128, 0, stream>>>(
      b.xt4, m, b.y4b, n, nps, st, b.row_part, rc.rb0, b.cull);
  FCPD_LAUNCH_CHECK();
  int32_t* list = b.row_flags + rc.r0;
  int32_t* count = b.flags_count + 1 + c;
  estep_row_combine_kernel<<<ceil_div((rc.r1 - rc.r0) * kCombineLanes, 256), 256, 0, stream>>>(
      b.row_part, splits, m, n, b.xt64, b.out, b.ystats, list, count, st, rc.r0, rc.r1);
  FCPD_LAUNCH_CHECK();
  estep_row_fallback_kernel<<<148, 256, 0, stream>>>(b.xt4, m, b.y4b, n, b.xt64, b.out,
                                                     b.ystats, list, count, st);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
