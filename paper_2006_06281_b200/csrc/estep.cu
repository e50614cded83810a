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
// Schedule (both passes): the work is the list of (own block, other tile)
// pairs — all of them, or the culled list (tile culling on spatially sorted
// points, list kernels below).  A persistent grid of exactly one CTA wave
// splits the list's POINTS evenly (stream-K): CTA g gets the contiguous
// range [g·P/G, (g+1)·P/G) of the P = 256·units point-units, cut into
// segments at block boundaries.  Every CTA therefore does the same work to
// within one point, independent of how culling thinned the list.  A segment
// (CTA g, block b) writes its fp64 partial sums to slot g + b (slots are
// strictly increasing along the schedule, so unique).  The CTA that
// completes a block's last segment (an arrival counter per block) sums the
// block's slots in CTA order and finalises the block: deterministic,
// bitwise reproducible, and no separate combine launch.

#include <cuda_runtime.h>
#include <math.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "estep.cuh"
#include "estep_device.cuh"

#ifndef FCPD_ROW_MINB
#define FCPD_ROW_MINB 12  // pass-2 CTAs per SM (80 registers: C4 pass 2 −5 % against 10)
#endif
namespace fcpd {

namespace {

constexpr int kTile = kTilePts;  // points staged in shared memory per step
constexpr float kPadCoord = 3.0e18f;  // padding point: t ≈ 1e37, 2^-t = 0
constexpr int kListThreads = 256;     // list kernels: one CTA per own block
static_assert(kListThreads == kTilePts, "list CTA: one thread per own point");
constexpr int kProbeTiles = 2;        // other-set tiles probed for the exact culling bound
constexpr int kFlush2 = 64;  // pass-2 fp32 run length (staged points; tools/gpu_flush.sh)
constexpr int64_t kMinPtsPerCta = 256;  // stream-K grid: dense point-units per CTA, at least (one chunk)
// Probe policy (speed only; any probe decision keeps the bound exact): probe
// a block when the tiles the box bound keeps but U = 0 would drop are ≥ 1/2
// of the kept ones; keep probing it every iteration while the probe drops
// ≥ 1/4 of them, else reconsider every 4th iteration.
constexpr float kProbeMinShare = 2.f;
constexpr float kProbePayShare = 4.f;
constexpr int kProbeRetry = 3;

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

// stream-K geometry over P point-units and G CTAs
__device__ __forceinline__ int64_t sk_start(int64_t g, int64_t G, int64_t P) { return g * P / G; }
__device__ __forceinline__ int64_t sk_owner(int64_t p, int64_t G, int64_t P) {
  return ((p + 1) * G - 1) / P;  // the CTA whose range holds point-unit p
}
// largest block b with off(b) ≤ u (u < total)
__device__ __forceinline__ int wl_block_of(const WorkList& wl, int64_t u) {
  if (wl.implicit) return static_cast<int>(u / wl.n_other);
  int lo = 0, hi = wl.n_blocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (wl.offset[mid] <= u) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Point index (in the other set) of list position e of block b: the units
// are upts()-point runs of consecutive points.
__device__ __forceinline__ int64_t wl_point(const WorkList& wl, int b, int64_t e) {
  const int64_t k = e >> wl.ushift;
  return (static_cast<int64_t>(wl.tile(b, k)) << wl.ushift) + (e - (k << wl.ushift));
}

// Centre and squared half-diagonal of the CTA's points' bounding box
// (scaled frame); blockDim ≤ 128.  Callers separate successive calls by a
// __syncthreads (the staging barrier).
struct BoxCentre {
  float3 c;
  float r2;
};
__device__ __forceinline__ BoxCentre cta_box_centre(float lx, float ly, float lz, float hx,
                                                    float hy, float hz) {
  __shared__ float red[6][4];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
    ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
    lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
    hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
    hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
    hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = lx;
    red[1][w] = ly;
    red[2][w] = lz;
    red[3][w] = hx;
    red[4][w] = hy;
    red[5][w] = hz;
  }
  __syncthreads();
  float r[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) r[k] = red[k][0];
  const int nw = blockDim.x >> 5;  // ≤ 4
  for (int i = 1; i < nw; ++i) {
#pragma unroll
    for (int k = 0; k < 3; ++k) r[k] = fminf(r[k], red[k][i]);
#pragma unroll
    for (int k = 3; k < 6; ++k) r[k] = fmaxf(r[k], red[k][i]);
  }
  BoxCentre b;
  if (!(r[0] <= r[3])) {  // no valid point
    b.c = make_float3(0.f, 0.f, 0.f);
    b.r2 = INFINITY;
    return b;
  }
  b.c = make_float3(0.5f * (r[0] + r[3]), 0.5f * (r[1] + r[4]), 0.5f * (r[2] + r[5]));
  const float ex = 0.5f * (r[3] - r[0]), ey = 0.5f * (r[4] - r[1]), ez = 0.5f * (r[5] - r[2]);
  b.r2 = ex * ex + ey * ey + ez * ez;
  return b;
}

__device__ __forceinline__ float2 ex2x2(float2 v) {
  return make_float2(ex2_approx(v.x), ex2_approx(v.y));
}

// 2^x on the FMA pipe for two lanes (the MUFU-bound pass 1 leaves its FP32
// pipe ~60 % idle): x = r + f with r = round(x) by the 1.5·2^23 trick and
// f ∈ [−½, ½]; 2^f by a degree-5 polynomial (max relative error 3.5e-7 in
// fp32 Horner; MUFU ex2.approx: ~2.4e-7); 2^r added to the exponent bits.
// x is clamped to ≥ −125 (smaller terms are < 2^-125 — the flush-to-zero
// MUFU returns 0 there; both are far below the column-total guard).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5·2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = __ffma2_rn(make_float2(0.0012915669940412045f, 0.0012915669940412045f), f,
                        make_float2(0.009668530896306038f, 0.009668530896306038f));
  p = __ffma2_rn(p, f, make_float2(0.055516887456178665f, 0.055516887456178665f));
  p = __ffma2_rn(p, f, make_float2(0.24022264778614044f, 0.24022264778614044f));
  p = __ffma2_rn(p, f, make_float2(0.6931464672088623f, 0.6931464672088623f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  // t's low mantissa bits hold r (two's complement); << 23 moves it to the exponent
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

}  // namespace

// ---------------------------------------------------------------------------
// Iteration-0 state (later iterations get theirs from the last step of the
// previous one, estep_scalars_for_next).
__global__ void init_state_kernel(IterState* st, double sigma2, double omega, int64_t m,
                                  int64_t n, int d) {
  st->omega = omega;
  st->m_all = m;
  st->n_all = n;
  st->dim = d;
  st->cull_pays = 0;
  // re-check every iteration when the pair work dwarfs the list kernels
  st->cull_recheck = static_cast<double>(m) * static_cast<double>(n) >= 2e9 ? 1 : kCullRecheck;
  estep_scalars_for_next(st, sigma2, 0);
  st->sigma2_e_last = st->sigma2_e;
}

// ---------------------------------------------------------------------------
// Block fix-up shared by both passes.  A block's segments come from the CTAs
// [g0, g1] of the stream-K range holding its point-units (those with a
// non-empty range); each bumps the block's arrival counter after writing its
// slot, and the one that arrives last sums the slots in CTA order.
struct SegRange {
  int64_t g0 = 0, g1 = -1;
  int count = 0;
};
__device__ __forceinline__ bool sk_empty(int64_t g, int64_t G, int64_t P) {
  // an empty range needs P < G (a range holds ⌊P/G⌋ or ⌈P/G⌉ units)
  return P < G && sk_start(g, G, P) == sk_start(g + 1, G, P);
}
__device__ __forceinline__ SegRange seg_range(const WorkList& wl, int64_t G, int64_t P, int b) {
  SegRange r;
  const int64_t ua = wl.off(b) << wl.ushift, ub = wl.off(b + 1) << wl.ushift;
  if (ua >= ub) return r;
  r.g0 = sk_owner(ua, G, P);
  r.g1 = sk_owner(ub - 1, G, P);
  if (P >= G) {
    r.count = static_cast<int>(r.g1 - r.g0 + 1);
  } else {
    for (int64_t g = r.g0; g <= r.g1; ++g) r.count += sk_empty(g, G, P) ? 0 : 1;
  }
  return r;
}
// Culling sessions use the culled list only when this iteration built one;
// otherwise every unit (counted into tiles_evaluated by CTA 0).
__device__ __forceinline__ WorkList resolve_list(WorkList wl, bool count = true) {
  if (wl.dyn_on && !*wl.dyn_on) {
    wl.implicit = 1;
    if (count && wl.implicit_counter && blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd(wl.implicit_counter, static_cast<unsigned long long>(wl.n_blocks) *
                                         static_cast<unsigned long long>(wl.n_other));
  }
  return wl;
}

// Pass-1 column finalisation (the block fix-up, and blocks a culled list
// left empty): b_n = −log2(Σ_m 2^{−t_mn} + c), Σ_m P_mn — or the exact
// fallback's queue when the mass is too small for the flush-to-zero fast
// path (flushed terms are < 2^-126 each: ≤ M·2^-126 in total; need ≤ 2^-50
// of the total).  Returns b as float, NaN when queued.
struct ColFix {
  int32_t* done;      // [col_blocks] arrival counters
  float4* y4b;        // .w ← b_n
  double* b2;
  double* pt1;        // optional
  int32_t* flag_list;
  float2* bminmax;    // optional (culling): per scene tile / sub-tile b range
  float2* sbminmax;
};
__device__ __forceinline__ float col_finalize(const ColFix& f, int64_t col, double sm, int64_t m,
                                              IterState* st) {
  const double c = exp2(st->log2c);  // 0 when ω = 0
  const double total = sm + c;
  if (!(total >= static_cast<double>(m) * 0x1p-76)) {
    const int slot = atomicAdd(&st->flag_count[0], 1);
    f.flag_list[slot] = static_cast<int32_t>(col);
    return NAN;  // the fallback writes b2 / pt1
  }
  const double b2 = -log2(total);
  f.b2[col] = b2;
  f.y4b[col].w = static_cast<float>(b2);
  if (f.pt1) f.pt1[col] = sm / total;
  return static_cast<float>(b2);
}

// Per scene tile and 32-column sub-tile: (min b, max b) for the pass-2
// list, kCols consecutive columns per thread.  Columns queued for the
// fallback (b unknown yet) count as +inf for the max and are left out of
// the min (no known b at all → −inf: no floor from that unit) — both
// conservative for the culling bounds.
template <int kCols>
__device__ __forceinline__ void col_b_ranges(const ColFix& f, int rb, int64_t n, float lo,
                                             float hi) {
  constexpr int kPerSub = kSubPts / kCols;  // threads per sub-tile
  const int t = threadIdx.x;
#pragma unroll
  for (int o = 1; o < kPerSub; o <<= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int64_t sub = static_cast<int64_t>(rb) * kSubPerTile + t / kPerSub;
  if (t % kPerSub == 0 && (sub << 5) < n)
    f.sbminmax[sub] = make_float2(lo == INFINITY ? -INFINITY : lo, hi);
#pragma unroll
  for (int o = kPerSub; o < 32; o <<= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ float2 red[8];
  if ((t & 31) == 0) red[t >> 5] = make_float2(lo, hi);
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      lo = fminf(lo, red[w].x);
      hi = fmaxf(hi, red[w].y);
    }
    f.bminmax[rb] = make_float2(lo == INFINITY ? -INFINITY : lo, hi);
  }
  __syncthreads();
}

// Pass-1 block fix-up: each column's sum over the block's slots in CTA
// order, finalisation, b ranges.
// ---------------------------------------------------------------------------
// Pass 1: per-column sums Σ_m 2^{−t_mn}.  Own block = 256 scene points
// (thread: column pair 2·tid, 2·tid+1); the staged tiles are model points.
//
// Two pair forms, chosen per segment (uniform across the CTA):
//  * centred (default where exact enough): with the block's box centre c,
//    u = y' − c, v = x' − c:  −t = 2u·v − |u|² − |v|², so a packed pair of
//    pairs costs FADD2 + 3 FFMA2 (+ FADD2 accumulate) and 2 MUFU.EX2;
//  * difference: −t = −‖y' − x'‖² (3 FADD2 + FMUL2 + 2 FFMA2), used when
//    the block's scaled radius makes the centred rounding (≈ 4ε·R²) too
//    large (kCentredMaxR2).
// f32x2 packing (FADD2/FMUL2/FFMA2, sm_100): each packed op evaluates two
// (m, n) pairs; each lane rounds like the scalar op.
// NC column pairs per thread; the CTA (128/NC threads) owns the 256-column
// block.  NC = 2 shares every staged model point's shared-memory operands
// between two packed column pairs (fewer LDS per pair).
// POLY of every 8 staged points take their ex2 on the FMA pipe (ex2_poly2)
// in the centred form: MUFU and FP32 balance at 2 (1/16·¾ = (4 + 8·¼)/128).
// MINB: CTAs per SM (NC = 2).  Large passes (C3, C4) run 32 (32 registers;
// the spills sit outside the inner loop): C4 pass 1 1.660 → 1.570 ms against
// 16, C3 3.14 → 3.00; on short ones (C1: < 2 staged chunks per CTA) 16 is
// the fastest (profiles/r2_pass_ab.txt).
template <int NC, int POLY, int MINB = 16>
__global__ void __launch_bounds__(128 / NC, NC == 2 ? MINB : 8)
    estep_col_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4,
                     int64_t n, IterState* __restrict__ st, WorkList wl_in,
                     double* __restrict__ seg, float centred_max_r2,
                     unsigned long long* form_pairs, uint64_t* stamps) {
  griddep_wait();
  constexpr int kThr = 128 / NC;  // threads
  constexpr int kCols = 2 * NC;   // columns per thread
  if (!st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0) stamps[4 * st->iter] = globaltimer();
  const WorkList wl = resolve_list(wl_in);
  // pair slots evaluated by form (centred, difference): thread 0's tally in
  // shared memory (no registers held across the pair loops)
  __shared__ unsigned long long form_tally[2];
  if (threadIdx.x == 0) form_tally[0] = form_tally[1] = 0ull;
  // staged model points as scalars, read as broadcast (.F32) FFMA2 operands
  // (as estep_row_kernel)
  __shared__ float4 xa[kTile];  // centred (vx, vy, vz, −|v|²) | diff (−x', −y', −z', ·)
  const float s = st->sx;
  const int64_t G = gridDim.x, g = blockIdx.x;
  const int64_t P = wl.off(wl.n_blocks) << wl.ushift;
  const int64_t p0 = sk_start(g, G, P), p1 = sk_start(g + 1, G, P);
  if (p0 >= p1) return;
  const int t = threadIdx.x;
  int rb = wl_block_of(wl, p0 >> wl.ushift);
  for (int64_t p = p0; p < p1;) {
    while ((wl.off(rb + 1) << wl.ushift) <= p) ++rb;
    const int64_t pe = min(p1, wl.off(rb + 1) << wl.ushift);
    const int64_t ob = wl.off(rb) << wl.ushift;  // first point-unit of block rb
    __syncthreads();  // previous segment's readers of the shared box/tiles are done
    // own columns of block rb
    const int64_t c0 = static_cast<int64_t>(rb) * kTile + kCols * t;
    float4 yv[kCols];
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int h = 0; h < kCols; ++h) {
      const int64_t c = c0 + h;
      yv[h] = c < n ? scale_pt(y4[c], s) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < n) {
        lo[0] = fminf(lo[0], yv[h].x), hi[0] = fmaxf(hi[0], yv[h].x);
        lo[1] = fminf(lo[1], yv[h].y), hi[1] = fmaxf(hi[1], yv[h].y);
        lo[2] = fminf(lo[2], yv[h].z), hi[2] = fmaxf(hi[2], yv[h].z);
      }
    }
    const BoxCentre bc = cta_box_centre(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const bool centred = bc.r2 <= centred_max_r2;  // < 0 → difference form only
    // per-thread operands per column pair: centred → 2u, −|u|²; diff → y'
    float2 ox[NC], oy[NC], oz[NC], on[NC];
#pragma unroll
    for (int q2 = 0; q2 < NC; ++q2) {
      if (centred) {
        float ux[2], uy[2], uz[2], q[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float4 y = yv[2 * q2 + h];
          ux[h] = __fsub_rn(y.x, bc.c.x);
          uy[h] = __fsub_rn(y.y, bc.c.y);
          uz[h] = __fsub_rn(y.z, bc.c.z);
          q[h] = __fmaf_rn(uz[h], uz[h], __fmaf_rn(uy[h], uy[h], __fmul_rn(ux[h], ux[h])));
        }
        ox[q2] = make_float2(2.f * ux[0], 2.f * ux[1]);
        oy[q2] = make_float2(2.f * uy[0], 2.f * uy[1]);
        oz[q2] = make_float2(2.f * uz[0], 2.f * uz[1]);
        on[q2] = make_float2(-q[0], -q[1]);
      } else {
        ox[q2] = make_float2(yv[2 * q2].x, yv[2 * q2 + 1].x);
        oy[q2] = make_float2(yv[2 * q2].y, yv[2 * q2 + 1].y);
        oz[q2] = make_float2(yv[2 * q2].z, yv[2 * q2 + 1].z);
        on[q2] = make_float2(0.f, 0.f);
      }
    }
    double d[kCols];
#pragma unroll
    for (int h = 0; h < kCols; ++h) d[h] = 0.0;
    for (int64_t q = p; q < pe;) {
      // stage the next ≤ 256 points of the block's list (gathered from its
      // units; points past m are padding)
      const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), pe - q));
      const int cnt8 = (cnt + 7) & ~7;
      __syncthreads();
      for (int i = t; i < cnt8; i += kThr) {
        const int64_t src = i < cnt ? wl_point(wl, rb, q + i - ob) : m;
        if (centred) {
          float4 v;
          if (src < m) {
            const float4 x = scale_pt(xt4[src], s);
            v = make_float4(__fsub_rn(x.x, bc.c.x), __fsub_rn(x.y, bc.c.y),
                            __fsub_rn(x.z, bc.c.z), 0.f);
            v.w = -__fmaf_rn(v.z, v.z, __fmaf_rn(v.y, v.y, __fmul_rn(v.x, v.x)));
          } else {  // padding row: −|v|² = −inf → 2^{−t} = 0 exactly
            v = make_float4(0.f, 0.f, 0.f, -INFINITY);
          }
          xa[i] = v;
        } else {
          const float4 v = src < m ? scale_pt(xt4[src], s)
                                   : make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
          xa[i] = make_float4(-v.x, -v.y, -v.z, 0.f);
        }
      }
      q += cnt;
      __syncthreads();
      float2 f[NC];
#pragma unroll
      for (int q2 = 0; q2 < NC; ++q2) f[q2] = make_float2(0.f, 0.f);
      if (centred) {
        for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 va = xa[j + u];
#pragma unroll
            for (int q2 = 0; q2 < NC; ++q2) {
              // 2u·v − |v|² = |u|² − t: the column's own 2^{−|u|²} is
              // factored out of its sum and applied once in fp64 (|u|² ≤ R²
              // ≤ 16, so the shifted terms stay in range)
              float2 e = __ffma2_rn(ox[q2], make_float2(va.x, va.x), make_float2(va.w, va.w));
              e = __ffma2_rn(oy[q2], make_float2(va.y, va.y), e);
              e = __ffma2_rn(oz[q2], make_float2(va.z, va.z), e);
              f[q2] = __fadd2_rn(f[q2], u < POLY ? ex2_poly2(e) : ex2x2(e));
            }
          }
        }
      } else {
        for (int j = 0; j < cnt8; j += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 va = xa[j + u];
#pragma unroll
            for (int q2 = 0; q2 < NC; ++q2) {
              const float2 dx = __fadd2_rn(ox[q2], make_float2(va.x, va.x));
              const float2 dy = __fadd2_rn(oy[q2], make_float2(va.y, va.y));
              const float2 dz = __fadd2_rn(oz[q2], make_float2(va.z, va.z));
              float2 tt = __fmul2_rn(dx, dx);
              tt = __ffma2_rn(dy, dy, tt);
              tt = __ffma2_rn(dz, dz, tt);
              f[q2] = __fadd2_rn(f[q2], ex2x2(make_float2(-tt.x, -tt.y)));
            }
          }
        }
      }
#pragma unroll
      for (int q2 = 0; q2 < NC; ++q2) {
        d[2 * q2] += static_cast<double>(f[q2].x);
        d[2 * q2 + 1] += static_cast<double>(f[q2].y);
      }
    }
    if (centred) {  // undo the factored-out 2^{|u|²}
#pragma unroll
      for (int q2 = 0; q2 < NC; ++q2) {
        d[2 * q2] *= exp2(static_cast<double>(on[q2].x));
        d[2 * q2 + 1] *= exp2(static_cast<double>(on[q2].y));
      }
    }
    double* out = seg + (g + rb) * kTile;
#pragma unroll
    for (int h = 0; h < kCols; ++h) out[kCols * t + h] = d[h];
    if (t == 0)
      form_tally[centred ? 0 : 1] += static_cast<unsigned long long>(pe - p) *
                                     static_cast<unsigned long long>(
                                         min(int64_t(kTile), n - int64_t(rb) * kTile));
    p = pe;
  }
  if (form_pairs && t == 0) {
    if (form_tally[0]) atomicAdd(form_pairs, form_tally[0]);
    if (form_tally[1]) atomicAdd(form_pairs + 1, form_tally[1]);
  }
}

// Exact column normaliser for flagged columns: warp per column, max-shifted
// log-sum-exp over all m in fp32 t_mn, fp64 accumulation.
// (run by the last CTA of the pass-1 combine: its warps take the queued
// columns in turn)
__device__ void col_fallback(const float4* __restrict__ xt4, int64_t m, float4* __restrict__ y4b,
                             double* __restrict__ b2_out, double* __restrict__ pt1,
                             const int32_t* __restrict__ flag_list, const IterState* st) {
  const int count = *reinterpret_cast<const volatile int32_t*>(&st->flag_count[0]);
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const float s = st->sx;
  const double log2c = st->log2c;
  for (int w = threadIdx.x >> 5; w < count; w += warps) {
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

// Where the pass-2 block fix-up puts a row's five sums (S0, Σw·y' (3), Σw·t
// in the scaled frame): single GPU → finalised (or queued for the exact
// fallback when the mass is too small for the flush-to-zero fast path);
// distributed → AoS row sums of this rank's columns for the reduce-scatter.
struct RowFix {
  int32_t* done;        // [row_blocks] arrival counters
  const double* xt64;
  RowOut out;
  YStats ys;
  int32_t* flag_list;
  double* aos;          // distributed: [m_pad][5] (then out/flag_list unused)
};
__device__ __forceinline__ void row_finalize(const RowFix& f, int64_t row, int64_t m, int64_t n,
                                             const double (&a)[5], IterState* st) {
  if (f.aos) {
#pragma unroll
    for (int k = 0; k < 5; ++k) f.aos[row * 5 + k] = a[k];
    return;
  }
  if (!(a[0] >= static_cast<double>(n) * 0x1p-76)) {
    const int slot = atomicAdd(&st->flag_count[1], 1);
    f.flag_list[slot] = static_cast<int32_t>(row);
    return;
  }
  finalize_row(row, m, log2(a[0]), a[0], a[1], a[2], a[3], a[4], f.xt64, derived_scale(st), f.out,
               f.ys, st);
}
// ---------------------------------------------------------------------------
// Pass 2: per-row sums over n: S0, Sy (3), SV.  Own block = 256 model points
// (thread: row pair 2·tid, 2·tid+1); the staged tiles are scene points.
//  * centred: L = (b − |u|²) − |v|² + 2u·v with u = y' − c, v = x' − c, and
//    the sums kept as Σw, Σw·u, Σw·|u|²; converted per segment in fp64:
//      Σw·y' = Σw·u + c·Σw,  Σw·t = Σw·|u|² + |v|²·Σw − 2v·Σw·u.
//    Per packed pair of pairs: 3 FFMA2 (L) + FADD2 + 4 FFMA2 (sums).
//  * difference: t = ‖y' − x'‖², L = b − t; sums Σw, Σw·y', Σw·t directly.
// MUFU and FP32 are co-bound (8 lane-ops per ex2); the staged scene values
// are broadcast (.F32) FFMA2 operands, which took the inner loop from 26.1
// to 22.7 cycles per 64 pairs per SMSP (tools/operand_bench.cu).
// NP row pairs per thread; the CTA (128/NP threads) owns the 256-row block.
// NP = 2 shares every staged scene point's operands between two packed row
// pairs (fewer register-operand reads per pair: −7.5 % per pair in
// tools/loopbench.cu).
template <int NP>
__global__ void __launch_bounds__(128 / NP, NP == 1 ? 8 : FCPD_ROW_MINB)
    estep_row_kernel(const float4* __restrict__ xt4, int64_t m, const float4* __restrict__ y4b,
                     int64_t n, IterState* __restrict__ st, WorkList wl_in,
                     double* __restrict__ seg /* [slot][5][256] */, float centred_max_r2,
                     int flush, unsigned long long* form_pairs) {
  griddep_wait();
  constexpr int kThr = 128 / NP;   // threads
  constexpr int kRows = 2 * NP;    // rows per thread
  if (!st->active) return;
  const WorkList wl = resolve_list(wl_in);
  // pair slots evaluated by form (centred, difference): thread 0's tally in
  // shared memory (no registers held across the pair loops)
  __shared__ unsigned long long form_tally[2];
  if (threadIdx.x == 0) form_tally[0] = form_tally[1] = 0ull;
  // staged scene points as scalars, read by the packed FFMA2s as broadcast
  // (.F32) operands: one LDS.128 (+ one LDS.32) per point and half the
  // register-operand traffic of duplicated (u,u) pairs (26.1 → 22.7 cycles
  // per 64 pairs per SMSP, tools/operand_bench.cu)
  __shared__ float4 ya[kTile];  // centred (ux, uy, uz, b − |u|²) | diff (y'x, y'y, y'z, b)
  __shared__ float yq[kTile];   // centred |u|²
  // fp64 tile accumulators in shared memory (thread-private slots,
  // [quantity][row][thread] → conflict-free): registers stay with the
  // packed pipeline
  __shared__ double acc_s[5][kRows][kThr];
  const float s = st->sx;
  const int64_t G = gridDim.x, g = blockIdx.x;
  const int64_t P = wl.off(wl.n_blocks) << wl.ushift;
  const int64_t p0 = sk_start(g, G, P), p1 = sk_start(g + 1, G, P);
  if (p0 >= p1) return;
  const float2 minus1 = make_float2(-1.f, -1.f);
  const int t = threadIdx.x;
  int rb = wl_block_of(wl, p0 >> wl.ushift);
  for (int64_t p = p0; p < p1;) {
    while ((wl.off(rb + 1) << wl.ushift) <= p) ++rb;
    const int64_t pe = min(p1, wl.off(rb + 1) << wl.ushift);
    const int64_t ob = wl.off(rb) << wl.ushift;  // first point-unit of block rb
    __syncthreads();  // previous segment's readers of the shared box/tiles are done
    const int64_t r0 = static_cast<int64_t>(rb) * kTile + kRows * t;
    float4 xv[kRows];
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int h = 0; h < kRows; ++h) {
      const int64_t r = r0 + h;
      xv[h] = r < m ? scale_pt(xt4[r], s) : make_float4(kPadCoord, kPadCoord, kPadCoord, 0.f);
      if (r < m) {
        lo[0] = fminf(lo[0], xv[h].x), hi[0] = fmaxf(hi[0], xv[h].x);
        lo[1] = fminf(lo[1], xv[h].y), hi[1] = fmaxf(hi[1], xv[h].y);
        lo[2] = fminf(lo[2], xv[h].z), hi[2] = fmaxf(hi[2], xv[h].z);
      }
    }
    const BoxCentre bc = cta_box_centre(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const bool centred = bc.r2 <= centred_max_r2;  // < 0 → difference form only
    // fp32 run length of the centred sums: the conversion to Σw·t cancels
    // terms of size R², so the rounding bound scales with run × R²; `flush`
    // is the run for the largest radius the form allows (R² = 16), and a
    // smaller block radius (the dense, large-σ² iterations) takes
    // proportionally longer runs, up to a whole staged chunk, under the same
    // bound
    int run = flush;
    if (centred)
      while (run < kTile && bc.r2 * static_cast<float>(2 * run) <= kCentredMaxR2 * flush) run *= 2;
    // per-thread operands per row pair: centred → 2v (and v, |v|² for the
    // conversion); diff → −x'
    float v[kRows][4];
    float2 ox[NP], oy[NP], oz[NP];
    if (centred) {
#pragma unroll
      for (int h = 0; h < kRows; ++h) {
        const bool ok = r0 + h < m;
        v[h][0] = ok ? __fsub_rn(xv[h].x, bc.c.x) : 0.f;
        v[h][1] = ok ? __fsub_rn(xv[h].y, bc.c.y) : 0.f;
        v[h][2] = ok ? __fsub_rn(xv[h].z, bc.c.z) : 0.f;
        v[h][3] = __fmaf_rn(v[h][2], v[h][2], __fmaf_rn(v[h][1], v[h][1], __fmul_rn(v[h][0], v[h][0])));
      }
#pragma unroll
      for (int q2 = 0; q2 < NP; ++q2) {
        ox[q2] = make_float2(2.f * v[2 * q2][0], 2.f * v[2 * q2 + 1][0]);
        oy[q2] = make_float2(2.f * v[2 * q2][1], 2.f * v[2 * q2 + 1][1]);
        oz[q2] = make_float2(2.f * v[2 * q2][2], 2.f * v[2 * q2 + 1][2]);
      }
    } else {
#pragma unroll
      for (int q2 = 0; q2 < NP; ++q2) {
        ox[q2] = make_float2(-xv[2 * q2].x, -xv[2 * q2 + 1].x);
        oy[q2] = make_float2(-xv[2 * q2].y, -xv[2 * q2 + 1].y);
        oz[q2] = make_float2(-xv[2 * q2].z, -xv[2 * q2 + 1].z);
      }
    }
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
      for (int h = 0; h < kRows; ++h) acc_s[k][h][t] = 0.0;
    for (int64_t q = p; q < pe;) {
      const int cnt = static_cast<int>(min(static_cast<int64_t>(kTile), pe - q));
      const int cnt8 = (cnt + 7) & ~7;
      __syncthreads();
      for (int i = t; i < cnt8; i += kThr) {
        const int64_t src = i < cnt ? wl_point(wl, rb, q + i - ob) : n;
        if (centred) {
          float4 u;
          float uq;
          if (src < n) {
            const float4 y = scale_pt(y4b[src], s);
            u = make_float4(__fsub_rn(y.x, bc.c.x), __fsub_rn(y.y, bc.c.y),
                            __fsub_rn(y.z, bc.c.z), 0.f);
            uq = __fmaf_rn(u.z, u.z, __fmaf_rn(u.y, u.y, __fmul_rn(u.x, u.x)));
            u.w = __fsub_rn(y.w, uq);  // b − |u|²
          } else {  // padding column: b = −inf → weight exactly 0
            u = make_float4(0.f, 0.f, 0.f, -INFINITY);
            uq = 0.f;
          }
          ya[i] = u;
          yq[i] = uq;
        } else {
          ya[i] = src < n ? scale_pt(y4b[src], s)
                          : make_float4(kPadCoord, kPadCoord, kPadCoord, -INFINITY);
        }
      }
      q += cnt;
      __syncthreads();
      float2 f0[NP], fx[NP], fy[NP], fz[NP], fv[NP];
#pragma unroll
      for (int q2 = 0; q2 < NP; ++q2)
        f0[q2] = fx[q2] = fy[q2] = fz[q2] = fv[q2] = make_float2(0.f, 0.f);
      // the fp32 sums go to fp64 every `flush` staged points (a power of
      // two) and at the end of the chunk: the centred form's conversion to
      // Σw·t cancels terms of size R², so the fp32 run length sets the
      // precision of the σ² terms (EStepPlan::flush2)
      auto flush_rows = [&]() {
#pragma unroll
        for (int q2 = 0; q2 < NP; ++q2) {
          const int h0 = 2 * q2, h1 = 2 * q2 + 1;
          acc_s[0][h0][t] += f0[q2].x;
          acc_s[0][h1][t] += f0[q2].y;
          acc_s[1][h0][t] += fx[q2].x;
          acc_s[1][h1][t] += fx[q2].y;
          acc_s[2][h0][t] += fy[q2].x;
          acc_s[2][h1][t] += fy[q2].y;
          acc_s[3][h0][t] += fz[q2].x;
          acc_s[3][h1][t] += fz[q2].y;
          acc_s[4][h0][t] += fv[q2].x;
          acc_s[4][h1][t] += fv[q2].y;
          f0[q2] = fx[q2] = fy[q2] = fz[q2] = fv[q2] = make_float2(0.f, 0.f);
        }
      };
      if (centred) {
        for (int j = 0; j < cnt8; j += 8) {
          if (j > 0 && (j & (run - 1)) == 0) flush_rows();  // uniform
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 A = ya[j + u];
            const float q = yq[j + u];
            const float2 Q = make_float2(q, q);
            const float2 Ux = make_float2(A.x, A.x), Uy = make_float2(A.y, A.y);
            const float2 Uz = make_float2(A.z, A.z), Bn = make_float2(A.w, A.w);
#pragma unroll
            for (int q2 = 0; q2 < NP; ++q2) {
              // b − |u|² + 2u·v = (b − t) + |v|²: the row's own 2^{|v|²} is
              // factored out of its sums and undone once in fp64 (|v|² ≤ 16)
              float2 L = __ffma2_rn(Ux, ox[q2], Bn);
              L = __ffma2_rn(Uy, oy[q2], L);
              L = __ffma2_rn(Uz, oz[q2], L);
              const float2 w = ex2x2(L);
              f0[q2] = __fadd2_rn(f0[q2], w);
              fx[q2] = __ffma2_rn(w, Ux, fx[q2]);
              fy[q2] = __ffma2_rn(w, Uy, fy[q2]);
              fz[q2] = __ffma2_rn(w, Uz, fz[q2]);
              fv[q2] = __ffma2_rn(w, Q, fv[q2]);
            }
          }
        }
      } else {
        for (int j = 0; j < cnt8; j += 8) {
          if (j > 0 && (j & (flush - 1)) == 0) flush_rows();  // uniform
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 A = ya[j + u];
            const float2 Yx = make_float2(A.x, A.x), Yy = make_float2(A.y, A.y);
            const float2 Yz = make_float2(A.z, A.z), Bn = make_float2(A.w, A.w);
#pragma unroll
            for (int q2 = 0; q2 < NP; ++q2) {
              const float2 ddx = __fadd2_rn(Yx, ox[q2]);
              const float2 ddy = __fadd2_rn(Yy, oy[q2]);
              const float2 ddz = __fadd2_rn(Yz, oz[q2]);
              float2 tt = __fmul2_rn(ddx, ddx);
              tt = __ffma2_rn(ddy, ddy, tt);
              tt = __ffma2_rn(ddz, ddz, tt);
              const float2 L = __ffma2_rn(tt, minus1, Bn);
              const float2 w = ex2x2(L);
              f0[q2] = __fadd2_rn(f0[q2], w);
              fx[q2] = __ffma2_rn(w, Yx, fx[q2]);
              fy[q2] = __ffma2_rn(w, Yy, fy[q2]);
              fz[q2] = __ffma2_rn(w, Yz, fz[q2]);
              fv[q2] = __ffma2_rn(w, tt, fv[q2]);
            }
          }
        }
      }
      flush_rows();
    }
    // segment out: S0, Σw·y', Σw·t per own row
    double* out = seg + (g + rb) * 5 * kTile;
#pragma unroll
    for (int h = 0; h < kRows; ++h) {
      const int li = kRows * t + h;
      double s0 = acc_s[0][h][t], s1 = acc_s[1][h][t], s2v = acc_s[2][h][t],
             s3 = acc_s[3][h][t], s4 = acc_s[4][h][t];
      if (centred) {
        const double vx = v[h][0], vy = v[h][1], vz = v[h][2], vq = v[h][3];
        const double sc = exp2(-vq);  // undo the factored-out 2^{|v|²}
        s0 *= sc;
        s1 *= sc;
        s2v *= sc;
        s3 *= sc;
        s4 *= sc;
        out[li] = s0;
        out[kTile + li] = s1 + static_cast<double>(bc.c.x) * s0;
        out[2 * kTile + li] = s2v + static_cast<double>(bc.c.y) * s0;
        out[3 * kTile + li] = s3 + static_cast<double>(bc.c.z) * s0;
        out[4 * kTile + li] = s4 + vq * s0 - 2.0 * (vx * s1 + vy * s2v + vz * s3);
      } else {
        out[li] = s0;
        out[kTile + li] = s1;
        out[2 * kTile + li] = s2v;
        out[3 * kTile + li] = s3;
        out[4 * kTile + li] = s4;
      }
    }
    if (t == 0)
      form_tally[centred ? 0 : 1] += static_cast<unsigned long long>(pe - p) *
                                     static_cast<unsigned long long>(
                                         min(int64_t(kTile), m - int64_t(rb) * kTile));
    p = pe;
  }
  if (form_pairs && t == 0) {
    if (form_tally[0]) atomicAdd(form_pairs, form_tally[0]);
    if (form_tally[1]) atomicAdd(form_pairs + 1, form_tally[1]);
  }
}

// ---------------------------------------------------------------------------
// Tile geometry and work lists for culling (points are k-d sorted by the
// engine, so 256-point tiles are spatially compact).

// per-tile and per-sub-tile axis-aligned boxes of the first three
// coordinates (unscaled): one CTA per 256-point tile, one warp per sub-tile
__global__ void tile_bbox_kernel(const float4* __restrict__ p, int64_t count,
                                 float4* __restrict__ lo, float4* __restrict__ hi,
                                 float4* __restrict__ slo, float4* __restrict__ shi,
                                 const IterState* __restrict__ st, uint64_t* stamps) {
  static_assert(kSubPts == 32, "one warp per sub-tile");
  griddep_wait();
  if (st && !st->active) return;
  // the first kernel of a culling session's iteration stamps its start
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0) stamps[4 * st->iter] = globaltimer();
  if (st && !st->cull_on) return;  // no lists this iteration: no x̃ boxes needed
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
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) red[k][warp] = v[k];
    const int64_t sub = static_cast<int64_t>(blockIdx.x) * kSubPerTile + warp;
    if (slo && (sub << 5) < count) {
      slo[sub] = make_float4(v[0], v[1], v[2], 0.f);
      shi[sub] = make_float4(v[3], v[4], v[5], 0.f);
    }
  }
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

// The last CTA of a list kernel turns the per-block counts (offset[b+1],
// and offset2[b+1] when given) into exclusive prefixes (in place), resets
// the done counter for the next graph replay and adds the total to the
// evaluated-pairs counter.
__device__ void scan_counts(int32_t* offset, int n_blocks, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  for (int base = 0; base < n_blocks; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int v = i < n_blocks ? __ldcg(offset + i + 1) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    if (i < n_blocks) offset[i + 1] = carry + before + v;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) offset[0] = 0;
}

__device__ bool last_cta_scan(int32_t* offset, int n_blocks, int32_t* done,
                              unsigned long long* counter) {
  __shared__ int is_last;
  __shared__ int wsum[32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  scan_counts(offset, n_blocks, wsum);
  if (threadIdx.x == 0) {
    *done = 0;
    if (counter) *counter += static_cast<unsigned long long>(offset[n_blocks]);
  }
  return true;
}

// CTA-wide reductions for the list kernels (kMax: max, else min; sums of
// small counts are exact in fp32).
template <bool kMax>
__device__ __forceinline__ float cta_reduce(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, w) : fminf(v, w);
  }
  __syncthreads();  // sh may still be read by a previous reduction
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = sh[0];
  for (int w = 1; w < kListThreads / 32; ++w) v = kMax ? fmaxf(v, sh[w]) : fminf(v, sh[w]);
  return v;
}
__device__ __forceinline__ float2 cta_sum2(float2 v, float2* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float2 r = sh[0];
  for (int w = 1; w < kListThreads / 32; ++w) r.x += sh[w].x, r.y += sh[w].y;
  return r;
}
__device__ __forceinline__ unsigned long long cta_min_u64(unsigned long long v,
                                                          unsigned long long* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = sh[0];
  for (int w = 1; w < kListThreads / 32; ++w) v = sh[w] < v ? sh[w] : v;
  return v;
}

// The kProbeTiles tiles of the other set whose box centres lie closest to
// the block's box centre (distinct; fewer when the other set has fewer).
__device__ __forceinline__ int probe_tiles(float4 lo, float4 hi, const float4* olo,
                                           const float4* ohi, int n_other, int* sel,
                                           unsigned long long* sh) {
  const float cx = 0.5f * (lo.x + hi.x), cy = 0.5f * (lo.y + hi.y), cz = 0.5f * (lo.z + hi.z);
  int count = 0;
  for (int r = 0; r < kProbeTiles && r < n_other; ++r) {
    unsigned long long best = ~0ull;
    for (int j = threadIdx.x; j < n_other; j += kListThreads) {
      bool taken = false;
      for (int q = 0; q < r; ++q) taken |= sel[q] == j;
      if (taken) continue;
      const float4 a = olo[j], b = ohi[j];
      const float dx = 0.5f * (a.x + b.x) - cx, dy = 0.5f * (a.y + b.y) - cy,
                  dz = 0.5f * (a.z + b.z) - cz;
      const float d2 = dx * dx + dy * dy + dz * dz;  // ≥ 0: bits order like the value
      const unsigned long long key =
          (static_cast<unsigned long long>(__float_as_uint(d2)) << 32) | static_cast<unsigned>(j);
      best = key < best ? key : best;
    }
    best = cta_min_u64(best, sh);
    sel[r] = static_cast<int>(best & 0xffffffffu);  // uniform across the CTA
    ++count;
  }
  return count;
}

// Append entry(j) for j < n, in order, to out[], skipping those that are
// −1 (entry(j) uniform per j); returns the count.
template <typename Entry>
__device__ __forceinline__ int cta_compact(int n, int32_t* out, int* wcount, Entry entry) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int count = 0;
  for (int j0 = 0; j0 < n; j0 += kListThreads) {
    const int j = j0 + threadIdx.x;
    const int32_t e = j < n ? entry(j) : -1;
    const bool k = e >= 0;
    const unsigned mask = __ballot_sync(0xffffffffu, k);
    __syncthreads();  // previous chunk's wcount readers are done
    if (lane == 0) wcount[warp] = __popc(mask);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < kListThreads / 32; ++w) {
      before += w < warp ? wcount[w] : 0;
      total += wcount[w];
    }
    if (k) out[count + before + __popc(mask & ((1u << lane) - 1))] = e;
    count += total;
  }
  return count;
}

// The units a list kernel visits after its tile-level screen: the units of
// the surviving 256-point tiles (a tile's units are boxes inside its box,
// so a bound that drops the tile drops them).  With few enough tiles the
// survivors are compacted into shared memory and only their units are
// visited; otherwise every unit is visited and screened by its tile.
constexpr int kMaxCandTiles = 4096;
struct UnitWalk {
  const int32_t* cand;  // surviving tiles (shared memory), or nullptr
  int n_work, upt, n_units;
  // unit of work item i, or −1 (past the end / screened out)
  template <typename TileIn>
  __device__ __forceinline__ int unit(int i, TileIn tile_in) const {
    if (cand) {
      const int u = cand[i / upt] * upt + i % upt;
      return u < n_units ? u : -1;
    }
    return tile_in(i / upt) ? i : -1;
  }
};
template <typename TileIn>
__device__ __forceinline__ UnitWalk unit_walk(int n_tiles, int upt, int n_units, int32_t* cand_s,
                                              int* wcount, TileIn tile_in) {
  UnitWalk w{nullptr, n_units, upt, n_units};
  if (n_tiles <= kMaxCandTiles) {
    const int nc = cta_compact(n_tiles, cand_s, wcount, [&](int j) { return tile_in(j) ? j : -1; });
    __syncthreads();  // publish cand_s
    w.cand = cand_s;
    w.n_work = nc * upt;
  }
  return w;
}

// Probe staging: candidate points centred on the own block's box centre,
// pair-interleaved for f32x2 math: pa[k] = (x_2k, x_2k+1, y_2k, y_2k+1),
// pb[k] = (z_2k, z_2k+1, q_2k, q_2k+1).
__device__ __forceinline__ void probe_stage(float4* pa, float4* pb, int i, float vx, float vy,
                                            float vz, float q) {
  float* fa = reinterpret_cast<float*>(pa) + (i >> 1) * 4 + (i & 1);
  float* fb = reinterpret_cast<float*>(pb) + (i >> 1) * 4 + (i & 1);
  fa[0] = vx;
  fa[2] = vy;
  fb[0] = vz;
  fb[2] = q;
}
// min (kMax: max) over the staged points of q_i + a·v_i: 3 FFMA2 per two
// points, four independent chains
template <bool kMax>
__device__ __forceinline__ float probe_scan(const float4* pa, const float4* pb, int pairs,
                                            float ax, float ay, float az) {
  const float2 X = make_float2(ax, ax), Y = make_float2(ay, ay), Z = make_float2(az, az);
  const float init = kMax ? -INFINITY : INFINITY;
  float r[4] = {init, init, init, init};
  for (int k = 0; k < pairs; k += 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 A = pa[k + h], B = pb[k + h];
      float2 d = __ffma2_rn(X, make_float2(A.x, A.y), make_float2(B.z, B.w));
      d = __ffma2_rn(Y, make_float2(A.z, A.w), d);
      d = __ffma2_rn(Z, make_float2(B.x, B.y), d);
      r[2 * h] = kMax ? fmaxf(r[2 * h], d.x) : fminf(r[2 * h], d.x);
      r[2 * h + 1] = kMax ? fmaxf(r[2 * h + 1], d.y) : fminf(r[2 * h + 1], d.y);
    }
  }
  return kMax ? fmaxf(fmaxf(r[0], r[1]), fmaxf(r[2], r[3]))
              : fminf(fminf(r[0], r[1]), fminf(r[2], r[3]));
}

// Pass-1 list, one CTA per scene block b.  Every column n of the block has
// total ≥ max(2^{−t_min(n)}, 2^{log2 c}); the bound uses U ≥ max_n
// min_m ‖y_n − x̃_m‖², the smaller of
//  * the box bound min over model sub-tiles j of maxdist²(b, j) (taken over
//    the sub-tiles of the tiles a first, tile-level bound keeps: the
//    minimising sub-tile always lies in one), and
//  * the probe: the exact nearest distance of every column to the points of
//    the kProbeTiles model tiles nearest the block (padded up by 2^-16),
// and model sub-tile j is dropped when s²·mindist²(b, j) > min(s²U, −log2 c)
// + margin (every pair term in it is then < 2^-margin of the column total).
__global__ void __launch_bounds__(kListThreads)
    col_list_kernel(CullInfo cull, const float4* __restrict__ xt4, int64_t m,
                    const float4* __restrict__ y4, int64_t n, int32_t* __restrict__ tiles,
                    int32_t* __restrict__ offset, int n_blocks, int32_t* __restrict__ done,
                    IterState* __restrict__ st) {
  griddep_wait();
  if (!st->active || !st->cull_on) return;
  __shared__ float4 pa[kProbeTiles * kTile / 2], pb[kProbeTiles * kTile / 2];
  __shared__ unsigned long long sh64[kListThreads / 32];
  __shared__ float shf[kListThreads / 32];
  __shared__ int sel[kProbeTiles];
  __shared__ int wcount[kListThreads / 32];
  __shared__ float2 sh2[kListThreads / 32];
  const float s2 = st->sx * st->sx;
  const int b = blockIdx.x;
  const float4 lo = cull.ylo[b], hi = cull.yhi[b];
  const float neg_log2c = static_cast<float>(-st->log2c);  // +inf when ω = 0
  // tile level: U_t ≥ U (box bound over whole tiles), then the probe; the
  // cut they give (≥ the final cut) screens the model tiles, and only the
  // survivors' sub-tiles are read below
  float ut = INFINITY, far = 0.f;
  for (int j = threadIdx.x; j < cull.n_xtiles; j += kListThreads) {
    const float4 jl = cull.xlo[j], jh = cull.xhi[j];
    ut = fminf(ut, box_maxdist2(lo, hi, jl, jh));
    far = fmaxf(far, box_mindist2(lo, hi, jl, jh));
  }
  ut = cta_reduce<false>(ut, shf);
  far = cta_reduce<true>(far, shf);
  // Probe only where it can pay (policy above, counted over tiles): the
  // tiles the box bound keeps but U = 0 would drop bound what the probe can
  // drop.
  bool useful = s2 * far > fminf(0.f, neg_log2c) + cull.margin1;
  float kept_box = 0.f;  // in sub-tiles
  useful = useful && cull.probe &&
           (!cull.probe_paid1 || cull.probe_paid1[b] || (st->iter & kProbeRetry) == 0);
  if (useful) {
    const float cut_box = fminf(s2 * ut, neg_log2c) + cull.margin1;
    const float cut_min = fminf(0.f, neg_log2c) + cull.margin1;
    float2 k = make_float2(0.f, 0.f);  // (kept, contested) tiles
    for (int j = threadIdx.x; j < cull.n_xtiles; j += kListThreads) {
      const float t = s2 * box_mindist2(lo, hi, cull.xlo[j], cull.xhi[j]);
      k.x += t <= cut_box ? 1.f : 0.f;
      k.y += t <= cut_box && t > cut_min ? 1.f : 0.f;
    }
    k = cta_sum2(k, sh2);
    kept_box = k.x * kSubPerTile;
    useful = k.y * kProbeMinShare >= k.x;
  }
  const int np = cull.probe && useful
                     ? probe_tiles(lo, hi, cull.xlo, cull.xhi, cull.n_xtiles, sel, sh64)
                     : 0;
  // exact nearest distance of every column to the probed points, in the
  // expanded form |u|² − 2u·v + |v|² about the block centre c
  const float cx = 0.5f * (lo.x + hi.x), cy = 0.5f * (lo.y + hi.y), cz = 0.5f * (lo.z + hi.z);
  float vmax = 0.f;  // max |v|² of the probed points
  for (int i = threadIdx.x; i < np * kTile; i += kListThreads) {
    const int64_t g = static_cast<int64_t>(sel[i / kTile]) * kTile + i % kTile;
    if (g < m) {
      const float4 x = xt4[g];
      const float vx = x.x - cx, vy = x.y - cy, vz = x.z - cz;
      const float q = vx * vx + vy * vy + vz * vz;
      vmax = fmaxf(vmax, q);
      probe_stage(pa, pb, i, vx, vy, vz, q);
    } else {
      probe_stage(pa, pb, i, 0.f, 0.f, 0.f, INFINITY);
    }
  }
  vmax = cta_reduce<true>(vmax, shf);  // (its barrier also publishes the staging)
  const int64_t c = static_cast<int64_t>(b) * kTile + threadIdx.x;
  float nn = -INFINITY;  // invalid column: neutral for the max
  if (c < n && np > 0) {
    const float4 y = y4[c];
    const float ux = y.x - cx, uy = y.y - cy, uz = y.z - cz;
    const float uq = ux * ux + uy * uy + uz * uz;
    nn = fmaxf(0.f, uq + probe_scan<false>(pa, pb, np * kTile / 2, -2.f * ux, -2.f * uy,
                                            -2.f * uz));
  }
  // pad for the rounding of the expanded form (≤ a few ε·(|u|² + |v|²))
  const float ex = hi.x - lo.x, ey = hi.y - lo.y, ez = hi.z - lo.z;
  const float h2 = 0.25f * (ex * ex + ey * ey + ez * ez);
  const float probe = cta_reduce<true>(nn, shf) * (1.f + 0x1p-16f) + 0x1p-20f * (h2 + vmax);
  float u = np > 0 ? fminf(ut, probe) : ut;
  const float cut_t = fminf(s2 * u, neg_log2c) + cull.margin1;
  auto tile_in = [&](int j) {
    return !(s2 * box_mindist2(lo, hi, cull.xlo[j], cull.xhi[j]) > cut_t);
  };
  __shared__ int32_t cand_s[kMaxCandTiles];
  const UnitWalk walk = unit_walk(cull.n_xtiles, kSubPerTile, cull.n_xsub, cand_s, wcount, tile_in);
  // the sub-tile box bound over the surviving tiles (the minimising sub-tile
  // lies in one of them)
  for (int i = threadIdx.x; i < walk.n_work; i += kListThreads) {
    const int sj = walk.unit(i, tile_in);
    if (sj >= 0) u = fminf(u, box_maxdist2(lo, hi, cull.sxlo[sj], cull.sxhi[sj]));
  }
  u = cta_reduce<false>(u, shf);
  const float cut = fminf(s2 * u, neg_log2c) + cull.margin1;
  // (cut ≤ cut_t: the kept units lie in the walk's tiles)
  const int count = cta_compact(
      walk.n_work, tiles + static_cast<int64_t>(b) * cull.n_xsub, wcount, [&](int i) {
        const int sj = walk.unit(i, tile_in);
        return sj >= 0 && !(s2 * box_mindist2(lo, hi, cull.sxlo[sj], cull.sxhi[sj]) > cut) ? sj
                                                                                          : -1;
      });
  if (threadIdx.x == 0) {
    offset[b + 1] = count;
    if (np > 0 && cull.probe_paid1)
      cull.probe_paid1[b] = (kept_box - count) * kProbePayShare >= kept_box;
  }
  last_cta_scan(offset, n_blocks, done, cull.counters);
}

// Pass-2 list, one CTA per model block b, over units of the scene (32-point
// sub-tiles: ulo/uhi/ubm, n_units).
// Every row m of the block has max_n L_mn ≥ L_lb, the larger of
//  * the box bound max over scene units j of (min b − s²·maxdist²(b, j))
//    (over the units of the tiles a first, tile-level bound keeps),
//  * the probe: min over the block's rows of the exact max of b_n − s²‖y_n −
//    x̃_m‖² over the kProbeTiles scene tiles nearest the block (less a
//    rounding slack);
// scene unit j is dropped when its largest possible L (max b − s²·mindist²)
// < L_lb − margin.  Its last CTA also decides whether the lists paid for
// themselves this iteration (IterState::cull_pays).
__global__ void __launch_bounds__(kListThreads)
    row_list_kernel(CullInfo cull, const float4* __restrict__ xt4, int64_t m,
                    const float4* __restrict__ y4b, int64_t n, int32_t* __restrict__ tiles,
                    int32_t* __restrict__ offset, int n_blocks, int32_t* __restrict__ done,
                    const float4* __restrict__ ulo, const float4* __restrict__ uhi,
                    const float2* __restrict__ ubm, int n_units,
                    IterState* __restrict__ st) {
  constexpr int unit_mult = 1;
  griddep_wait();
  if (!st->active || !st->cull_on) return;
  __shared__ float4 pa[kProbeTiles * kTile / 2], pb[kProbeTiles * kTile / 2];
  __shared__ unsigned long long sh64[kListThreads / 32];
  __shared__ float shf[kListThreads / 32];
  __shared__ int sel[kProbeTiles];
  __shared__ int wcount[kListThreads / 32];
  __shared__ float2 sh2[kListThreads / 32];
  const float s2 = st->sx * st->sx;
  const int b = blockIdx.x;
  const float4 lo = cull.xlo[b], hi = cull.xhi[b];  // (pass 2: the model block)
  const int upt = kSubPerTile / unit_mult;  // units per scene tile (8, or 1: whole tiles)
  // a scene tile's largest possible L (its units' are no larger)
  auto tile_top = [&](int j) {
    return cull.bminmax[j].y - s2 * box_mindist2(lo, hi, cull.ylo[j], cull.yhi[j]);
  };
  float floor_l = -INFINITY, kept_box = 0.f;
  float floor_t = -INFINITY;  // tile-level floor (≤ floor_l): screens the tiles
  auto tile_in = [&](int j) { return !cull.enabled || !(tile_top(j) < floor_t); };
  __shared__ int32_t cand_s[kMaxCandTiles];
  UnitWalk walk{nullptr, n_units, upt, n_units};  // culling off: every unit
  int np = 0;
  if (cull.enabled) {
    float lt = -INFINITY, lmin = INFINITY;
    for (int j = threadIdx.x; j < cull.n_ytiles; j += kListThreads) {
      const float4 jl = cull.ylo[j], jh = cull.yhi[j];
      const float2 bm = cull.bminmax[j];
      lt = fmaxf(lt, bm.x - s2 * box_maxdist2(lo, hi, jl, jh));
      lmin = fminf(lmin, bm.y - s2 * box_mindist2(lo, hi, jl, jh));
    }
    lt = cta_reduce<true>(lt, shf);
    lmin = cta_reduce<false>(lmin, shf);
    float l = lt;
    // L ≤ 0, so a tile can only be dropped if its bound is below −margin;
    // probe policy as in pass 1, with L_lb = 0 as the optimistic bound
    bool useful = lmin < -cull.margin2;
    useful = useful && cull.probe &&
             (!cull.probe_paid2 || cull.probe_paid2[b] || (st->iter & kProbeRetry) == 0);
    if (useful) {  // counted over tiles
      const float floor_box = lt - cull.margin2;
      float2 k = make_float2(0.f, 0.f);
      for (int j = threadIdx.x; j < cull.n_ytiles; j += kListThreads) {
        const float v = tile_top(j);
        k.x += v >= floor_box ? 1.f : 0.f;
        k.y += v >= floor_box && v < -cull.margin2 ? 1.f : 0.f;
      }
      k = cta_sum2(k, sh2);
      kept_box = k.x * upt;
      useful = k.y * kProbeMinShare >= k.x;
    }
    np = cull.probe && useful
             ? probe_tiles(lo, hi, cull.ylo, cull.yhi, cull.n_ytiles, sel, sh64)
             : 0;
    // exact max over the probed columns of b_n − s²‖y_n − x̃_m‖² for every
    // row, expanded about the block centre c: (b − s²|v|²) + 2s²u·v − s²|u|²
    const float cx = 0.5f * (lo.x + hi.x), cy = 0.5f * (lo.y + hi.y),
                cz = 0.5f * (lo.z + hi.z);
    float vmax = 0.f;
    for (int i = threadIdx.x; i < np * kTile; i += kListThreads) {
      const int64_t g = static_cast<int64_t>(sel[i / kTile]) * kTile + i % kTile;
      if (g < n) {
        const float4 y = y4b[g];
        const float vx = y.x - cx, vy = y.y - cy, vz = y.z - cz;
        const float q = vx * vx + vy * vy + vz * vz;
        vmax = fmaxf(vmax, q);
        probe_stage(pa, pb, i, vx, vy, vz, y.w - s2 * q);
      } else {
        probe_stage(pa, pb, i, 0.f, 0.f, 0.f, -INFINITY);
      }
    }
    vmax = cta_reduce<true>(vmax, shf);
    const int64_t r = static_cast<int64_t>(b) * kTile + threadIdx.x;
    float best = INFINITY;  // invalid row: neutral for the min
    if (r < m && np > 0) {
      const float4 x = xt4[r];
      const float ux = x.x - cx, uy = x.y - cy, uz = x.z - cz;
      const float uq = ux * ux + uy * uy + uz * uz;
      const float t2 = 2.f * s2;
      best = probe_scan<true>(pa, pb, np * kTile / 2, t2 * ux, t2 * uy, t2 * uz) - s2 * uq;
    }
    const float probe = cta_reduce<false>(best, shf);
    const float ex = hi.x - lo.x, ey = hi.y - lo.y, ez = hi.z - lo.z;
    const float h2 = 0.25f * (ex * ex + ey * ey + ez * ez);
    // rounding slack of the fp32 bound (expanded form: ≲ a few ε·s²(|u|² + |v|²))
    if (np > 0) l = fmaxf(l, probe - 1e-3f - 1e-5f * fabsf(probe) - 0x1p-20f * s2 * (h2 + vmax));
    // the tile-level floor screens the scene tiles; the unit box bound over
    // the survivors (the maximising unit lies in one of them) tightens it
    floor_t = l - cull.margin2;
    walk = unit_walk(cull.n_ytiles, upt, n_units, cand_s, wcount, tile_in);
    for (int i = threadIdx.x; i < walk.n_work; i += kListThreads) {
      const int u = walk.unit(i, tile_in);
      if (u >= 0) l = fmaxf(l, ubm[u].x - s2 * box_maxdist2(lo, hi, ulo[u], uhi[u]));
    }
    l = cta_reduce<true>(l, shf);
    floor_l = l - cull.margin2;
  }
  // (floor_l ≥ floor_t: the kept units lie in the walk's tiles)
  const int count = cta_compact(
      walk.n_work, tiles + static_cast<int64_t>(b) * n_units, wcount, [&](int i) {
        const int u = walk.unit(i, tile_in);
        return u >= 0 && (!cull.enabled ||
                          !(ubm[u].y - s2 * box_mindist2(lo, hi, ulo[u], uhi[u]) < floor_l))
                   ? u
                   : -1;
      });
  if (threadIdx.x == 0) {
    offset[b + 1] = count;
    if (np > 0 && cull.probe_paid2)
      cull.probe_paid2[b] = (kept_box - count) * kProbePayShare >= kept_box;
  }
  if (last_cta_scan(offset, n_blocks, done, cull.counters ? cull.counters + 1 : nullptr) &&
      threadIdx.x == 0) {
    // the next iteration builds lists again if these dropped any unit (σ²
    // only falls, so a culling that starts to bite soon pays); otherwise
    // every kCullRecheck-th iteration
    const double kept1 = static_cast<double>(cull.wl1_offset[cull.n_ytiles]);
    const double kept2 = static_cast<double>(offset[n_blocks]);
    st->cull_pays = kept1 < kCullKeepFrac * static_cast<double>(cull.wl1_units) ||
                    kept2 < kCullKeepFrac * static_cast<double>(cull.wl2_units);
  }
}

// Exact row accumulation for flagged rows (tiny mass): warp per row,
// max-shifted, fp64 accumulation.
// (run by the last CTA of the pass-2 combine)
__device__ void row_fallback(const float4* __restrict__ xt4, int64_t m,
                             const float4* __restrict__ y4b, int64_t n,
                             const double* __restrict__ xt64, const RowOut& out, const YStats& ys,
                             const int32_t* __restrict__ flag_list, IterState* st) {
  const int count = *reinterpret_cast<const volatile int32_t*>(&st->flag_count[1]);
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const float s = st->sx;
  for (int w = threadIdx.x >> 5; w < count; w += warps) {
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
// Combines: one thread per column (pass 1) / row (pass 2), one CTA per
// 256-point block.  A point's segment slots are summed in CTA order with
// kCombineBatch independent loads in flight (skipped slots add +0.0, which
// leaves a sum of non-negative terms unchanged bit for bit), then finalised.
// The combine's last CTA runs the exact fallback of everything queued.
constexpr int kCombineBatch = 8;

__device__ __forceinline__ bool last_cta(int32_t* done) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  if (threadIdx.x == 0) *done = 0;  // self-resetting for the next replay
  return true;
}

// Pass-1 combine: b_n / Σ_m P_mn or the fallback queue, the tile's b ranges
// (culling), then (last CTA) the exact fallback of the queued columns.
__global__ void __launch_bounds__(kTile)
    estep_col_combine_kernel(const double* __restrict__ seg, WorkList wl_in, int G, int64_t m,
                             int64_t n, ColFix f, const float4* __restrict__ xt4,
                             IterState* __restrict__ st, int32_t* __restrict__ done) {
  griddep_wait();
  if (!st->active) return;
  const WorkList wl = resolve_list(wl_in, false);
  const int64_t P = wl.off(wl.n_blocks) << wl.ushift;
  const int b = blockIdx.x, li = threadIdx.x;
  const int64_t col = static_cast<int64_t>(b) * kTile + li;
  const SegRange sr = seg_range(wl, G, P, b);
  double sm = 0.0;
  for (int64_t g = sr.g0; g <= sr.g1; g += kCombineBatch) {
    double v[kCombineBatch];
#pragma unroll
    for (int j = 0; j < kCombineBatch; ++j)
      v[j] = g + j <= sr.g1 && !sk_empty(g + j, G, P) ? __ldcg(seg + (g + j + b) * kTile + li)
                                                       : 0.0;
#pragma unroll
    for (int j = 0; j < kCombineBatch; ++j) sm += v[j];
  }
  float lo = INFINITY, hi = -INFINITY;
  if (col < n) {
    const float bv = col_finalize(f, col, sm, m, st);
    if (bv == bv) {
      lo = bv;
      hi = bv;
    } else {
      hi = INFINITY;
    }
  }
  if (f.bminmax) col_b_ranges<1>(f, b, n, lo, hi);
  if (last_cta(done)) col_fallback(xt4, m, f.y4b, f.b2, f.pt1, f.flag_list, st);
}

// Pass-2 combine: finalised rows (or the fallback queue), or AoS row sums
// of the local columns (distributed); then (last CTA, single GPU) the exact
// fallback of the queued rows.
__global__ void __launch_bounds__(kTile)
    estep_row_combine_kernel(const double* __restrict__ seg, WorkList wl_in, int G, int64_t m,
                             int64_t n, RowFix f, const float4* __restrict__ xt4,
                             const float4* __restrict__ y4b, IterState* __restrict__ st,
                             int32_t* __restrict__ done) {
  griddep_wait();
  if (!st->active) return;
  const WorkList wl = resolve_list(wl_in, false);
  const int64_t P = wl.off(wl.n_blocks) << wl.ushift;
  const int b = blockIdx.x, li = threadIdx.x;
  const int64_t row = static_cast<int64_t>(b) * kTile + li;
  const SegRange sr = seg_range(wl, G, P, b);
  double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t g = sr.g0; g <= sr.g1; g += kCombineBatch) {
    double v[kCombineBatch][5];
#pragma unroll
    for (int j = 0; j < kCombineBatch; ++j) {
      const bool live = g + j <= sr.g1 && !sk_empty(g + j, G, P);
      const double* sp = seg + (g + j + b) * 5 * kTile + li;
#pragma unroll
      for (int k = 0; k < 5; ++k) v[j][k] = live ? __ldcg(sp + k * kTile) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kCombineBatch; ++j)
#pragma unroll
      for (int k = 0; k < 5; ++k) a[k] += v[j][k];
  }
  if (row < m) row_finalize(f, row, m, n, a, st);
  if (!f.aos && last_cta(done))
    row_fallback(xt4, m, y4b, n, f.xt64, f.out, f.ys, f.flag_list, st);
}

// ---------------------------------------------------------------------------
// Host-side launchers.

EStepPlan make_estep_plan(int64_t m, int64_t n, int sm_count) {
  EStepPlan p;
  if (const char* e = std::getenv("FCPD_ESTEP_FORM")) p.centred = std::strcmp(e, "diff") != 0;
  p.centred_max_r2 = p.centred ? kCentredMaxR2 : -1.f;
  if (const char* e = std::getenv("FCPD_CENTRED_MAX_R2"))  // precision/speed study
    p.centred_max_r2 = p.centred ? static_cast<float>(std::atof(e)) : -1.f;
  int occ_col = 0, occ_row = 0;
  // two column pairs per thread pay on large passes (fewer shared-memory
  // loads per pair); small ones (C0: 64 tile pairs) are latency-bound and
  // prefer more, lighter CTAs
  p.col_pairs = ceil_div(m, kTile) * ceil_div(n, kTile) >= 1024 ? 2 : 1;
  if (const char* e = std::getenv("FCPD_COL_PAIRS")) p.col_pairs = std::atoi(e) == 1 ? 1 : 2;
  if (const char* e = std::getenv("FCPD_EX2_POLY")) p.ex2_poly = std::max(0, std::min(3, std::atoi(e)));
  // 32 CTAs per SM where each still gets ≥ 8 staged 256-point chunks of the
  // dense pass (point-units of the implicit list over 32·SMs CTAs)
  {
    const int64_t units = static_cast<int64_t>(ceil_div(n, kTile)) * ceil_div(m, kSubPts) * kSubPts;
    p.col_minb = units / (static_cast<int64_t>(sm_count) * 32) >= 8 * kTile ? 32 : 16;
    if (const char* e = std::getenv("FCPD_COL_MINB")) p.col_minb = std::atoi(e) == 32 ? 32 : 16;
  }
  if (p.col_pairs == 2 && p.col_minb == 32)
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_col, estep_col_kernel<2, 0, 32>, 64, 0));
  else if (p.col_pairs == 2)
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_col, estep_col_kernel<2, 0>, 64, 0));
  else
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_col, estep_col_kernel<1, 0>, 128, 0));
  if (const char* e = std::getenv("FCPD_ROW_PAIRS")) p.row_pairs = std::atoi(e) == 1 ? 1 : 2;
  if (p.row_pairs == 2)
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_row, estep_row_kernel<2>, 64, 0));
  else
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_row, estep_row_kernel<1>, 128, 0));
  p.col_blocks = static_cast<int>(ceil_div(n, kTile));
  p.row_blocks = static_cast<int>(ceil_div(m, kTile));
  // One wave of CTAs, but at least kMinPtsPerCta point-units of the dense
  // pass per CTA: on small passes (C0: 8 blocks × 2000 points) a full wave
  // leaves each CTA a few points and each block's fix-up a long chain of
  // segment slots to sum.
  int64_t min_pts = kMinPtsPerCta;
  if (const char* e = std::getenv("FCPD_ESTEP_MIN_PTS")) min_pts = std::max<int64_t>(1, std::atoll(e));
  auto grid_for = [&](int64_t pts, int occ) {
    const int64_t full = static_cast<int64_t>(sm_count) * std::max(occ, 1);
    return static_cast<int>(std::min(full, std::max<int64_t>(sm_count, ceil_div(pts, min_pts))));
  };
  p.col_grid = grid_for(p.col_blocks * ceil_div(m, kSubPts) * kSubPts, occ_col);
  p.row_grid = grid_for(p.row_blocks * ceil_div(n, kSubPts) * kSubPts, occ_row);
  // fp32 run length of the pass-2 sums before they go to fp64
  auto flush_env = [](const char* name, int def) {
    const char* e = std::getenv(name);
    const int v = e ? std::atoi(e) : def;
    int f = 8;  // a power of two in [8, 256]
    while (f < kTile && 2 * f <= v) f *= 2;
    return f;
  };
  p.flush2 = flush_env("FCPD_FLUSH2", kFlush2);
  return p;
}

namespace {
// A culling session's lists are used only in iterations that build them
// (IterState::cull_on); the implicit fallback counts its units.
WorkList pass1_list(const EStepPlan& p, const EStepBuffers& b, int64_t m, const IterState* st) {
  WorkList wl;
  wl.implicit = b.cull.enabled ? 0 : 1;
  wl.n_blocks = p.col_blocks;
  wl.n_other = static_cast<int>(ceil_div(m, kSubPts));
  wl.tiles = b.wl1.tiles;
  wl.offset = b.wl1.offset;
  if (b.cull.enabled) {
    wl.dyn_on = &st->cull_on;
    wl.implicit_counter = b.cull.counters;
  }
  return wl;
}
WorkList pass2_list(const EStepPlan& p, const EStepBuffers& b, int64_t n, const IterState* st) {
  WorkList wl;
  wl.implicit = b.cull.enabled ? 0 : 1;
  wl.n_blocks = p.row_blocks;
  wl.ushift = 5;
  static_assert(kSubPts == 1 << 5, "unit shift");
  wl.n_other = static_cast<int>(ceil_div(n, kSubPts));
  wl.tiles = b.wl2.tiles;
  wl.offset = b.wl2.offset;
  if (b.cull.enabled) {
    wl.dyn_on = &st->cull_on;
    wl.implicit_counter = b.cull.counters ? b.cull.counters + 1 : nullptr;
  }
  return wl;
}
ColFix col_fix(const EStepBuffers& b) {
  return ColFix{b.col_done, b.y4b, b.b2, b.pt1, b.col_flags,
                b.cull.enabled ? b.cullw.bminmax : nullptr, b.cullw.sbminmax};
}
RowFix row_fix(const EStepBuffers& b) {
  return RowFix{b.row_done, b.xt64, b.out, b.ystats, b.row_flags, b.row_aos};
}
}  // namespace

int estep_kernels(bool culling, bool) {
  // pass 1 + its combine + pass 2 + its combine (the combines also run the
  // exact fallbacks and the b ranges); culling adds the x̃ tile boxes and the
  // two list kernels (launched every iteration; they return at once when the
  // iteration builds no lists)
  return 4 + (culling ? 3 : 0);
}

void launch_init_state(IterState* st, double sigma2, double omega, int64_t m, int64_t n_global,
                       int d, cudaStream_t stream) {
  init_state_kernel<<<1, 1, 0, stream>>>(st, sigma2, omega, m, n_global, d);
  FCPD_LAUNCH_CHECK();
}

void launch_tile_bbox(const float4* pts, int64_t count, float4* lo, float4* hi, float4* slo,
                      float4* shi, const IterState* st, cudaStream_t stream) {
  launch_pdl(tile_bbox_kernel, dim3(ceil_div(count, kTile)), dim3(kTile), 0, stream, pts, count, lo,
             hi, slo, shi, st, static_cast<uint64_t*>(nullptr));
  FCPD_LAUNCH_CHECK();
}

// Pass 1 (column normalisers): with culling, the model-tile boxes of this
// iteration's x̃ and the pass-1 work list before it; the column fallback
// after.  Scene-tile b ranges are written by the pass-1 block fix-up.
void launch_estep_pass1(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream) {
  const CullInfo& cu = b.cull;
  const WorkList wl = pass1_list(p, b, m, st);
  const ColFix fix = col_fix(b);
  unsigned long long* forms = cu.counters ? cu.counters + 2 : nullptr;
  if (cu.enabled) {
    // the first kernel of the iteration stamps its start
    launch_pdl(tile_bbox_kernel, dim3(ceil_div(m, kTile)), dim3(kTile), 0, stream, b.xt4, m,
               b.cullw.xlo, b.cullw.xhi, b.cullw.sxlo, b.cullw.sxhi,
               static_cast<const IterState*>(st), b.stamps);
    FCPD_LAUNCH_CHECK();
    launch_pdl(col_list_kernel, dim3(p.col_blocks), dim3(kListThreads), 0, stream, cu, b.xt4, m,
               b.y4b, n, b.wl1.tiles, b.wl1.offset, p.col_blocks, b.wl1.done, st);
    FCPD_LAUNCH_CHECK();
  }
  uint64_t* stamps = cu.enabled ? nullptr : b.stamps;
  auto col = [&](auto kernel, int threads) {
    launch_pdl(kernel, dim3(p.col_grid), dim3(threads), 0, stream, b.xt4, m,
               static_cast<const float4*>(b.y4b), n, st, wl, b.col_seg, p.centred_max_r2, forms,
               stamps);
  };
  if (p.col_pairs == 2 && p.col_minb == 32) {
    switch (p.ex2_poly) {
      case 1: col(estep_col_kernel<2, 1, 32>, 64); break;
      case 2: col(estep_col_kernel<2, 2, 32>, 64); break;
      case 3: col(estep_col_kernel<2, 3, 32>, 64); break;
      default: col(estep_col_kernel<2, 0, 32>, 64); break;
    }
  } else if (p.col_pairs == 2) {
    switch (p.ex2_poly) {
      case 1: col(estep_col_kernel<2, 1>, 64); break;
      case 2: col(estep_col_kernel<2, 2>, 64); break;
      case 3: col(estep_col_kernel<2, 3>, 64); break;
      default: col(estep_col_kernel<2, 0>, 64); break;
    }
  } else {
    col(estep_col_kernel<1, 0>, 128);
  }
  FCPD_LAUNCH_CHECK();
  launch_pdl(estep_col_combine_kernel, dim3(p.col_blocks), dim3(kTile), 0, stream,
             static_cast<const double*>(b.col_seg), wl, p.col_grid, m, n, fix, b.xt4, st,
             b.col_done);
  FCPD_LAUNCH_CHECK();
}

// Pass 2: the work list (culling), the row accumulation with its block
// fix-up (finalised rows, or AoS sums when distributed) and, on one GPU, the
// exact fallback of the rows the fix-up queued.
void launch_estep_pass2(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream) {
  const CullInfo& cu = b.cull;
  const WorkList wl = pass2_list(p, b, n, st);
  const RowFix fix = row_fix(b);
  unsigned long long* forms = cu.counters ? cu.counters + 4 : nullptr;
  if (cu.enabled) {
    launch_pdl(row_list_kernel, dim3(p.row_blocks), dim3(kListThreads), 0, stream, cu, b.xt4, m,
               static_cast<const float4*>(b.y4b), n, b.wl2.tiles, b.wl2.offset, p.row_blocks,
               b.wl2.done, static_cast<const float4*>(cu.sylo),
               static_cast<const float4*>(cu.syhi), static_cast<const float2*>(cu.sbminmax),
               wl.n_other, st);
    FCPD_LAUNCH_CHECK();
  }
  if (p.row_pairs == 2)
    launch_pdl(estep_row_kernel<2>, dim3(p.row_grid), dim3(64), 0, stream, b.xt4, m,
               static_cast<const float4*>(b.y4b), n, st, wl, b.row_seg, p.centred_max_r2,
               p.flush2, forms);
  else
    launch_pdl(estep_row_kernel<1>, dim3(p.row_grid), dim3(128), 0, stream, b.xt4, m,
               static_cast<const float4*>(b.y4b), n, st, wl, b.row_seg, p.centred_max_r2,
               p.flush2, forms);
  FCPD_LAUNCH_CHECK();
  launch_pdl(estep_row_combine_kernel, dim3(p.row_blocks), dim3(kTile), 0, stream,
             static_cast<const double*>(b.row_seg), wl, p.row_grid, m, n, fix, b.xt4,
             static_cast<const float4*>(b.y4b), st, b.row_done);
  FCPD_LAUNCH_CHECK();
}

void launch_estep(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                  IterState* st, cudaStream_t stream, cudaEvent_t mid) {
  launch_estep_pass1(p, b, m, n, st, stream);
  if (mid) FCPD_CUDA(cudaEventRecord(mid, stream));
  launch_estep_pass2(p, b, m, n, st, stream);
}

}  // namespace fcpd
