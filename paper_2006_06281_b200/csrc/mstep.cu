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
// makes both passes fully coalesced single reads of HBM.  The kernel is
// stream-K: a persistent grid (one wave of resident CTAs) splits the
// (row × 1024-column block) units evenly, so there is no tail wave and each
// CTA emits one partial per column block it touched.  fp32 products, fp32
// accumulation over 16-row groups, fp64 above that, and a fixed-order fp64
// reduction over partials (bitwise reproducible).
//
// σ² uses the cancellation-free per-row form: with
// Δ̄_m = (P̃Y)_m − x̃old_m, V_m = Σ_n P̃_mn‖y_n − x̃old_m‖², δ = x̃new − x̃old,
//     σ² = Σ_m [V_m − 2 δ_m·Δ̄_m + ‖δ_m‖²] / (D M),
// algebraically identical to the reference trace form because rows of P̃
// sum to one.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "mstep.cuh"

namespace fcpd {

namespace {
constexpr int kRowGroup = 16;  // rows per fp32 sub-accumulation / loads in flight

struct SkGeom {
  int64_t rows, cols4, units;
  int grid, kmax;
  int trunc;  // ColsumPlan::trunc
};

// The geometry actually streamed this iteration: with spectral truncation
// the eigenvector axis (columns of Q, rows of Qᵀ) stops at st->keff.  Every
// kernel of one stream (colsum, reduction) derives the same geometry.
__device__ __forceinline__ SkGeom sk_eff(SkGeom g, const IterState* st) {
  if (!g.trunc || !st) return g;
  const int64_t keff = st->keff;
  if (g.trunc == 1) {
    g.cols4 = min(g.cols4, (keff + 3) / 4);
    g.units = (g.cols4 + kColsumThreads - 1) / kColsumThreads * g.rows;
  } else {
    const int64_t col_blocks = g.units / g.rows;
    g.rows = min(g.rows, keff);
    g.units = col_blocks * g.rows;
  }
  return g;
}

__host__ __device__ __forceinline__ int64_t sk_begin(const SkGeom& g, int64_t cta) {
  return cta * g.units / g.grid;
}
// CTA owning work unit u: the g with begin(g) ≤ u < begin(g+1)
__device__ __forceinline__ int64_t sk_owner(const SkGeom& g, int64_t u) {
  return ((u + 1) * g.grid - 1) / g.units;
}

// Fixed-order sum of the partials covering column c.
__device__ __forceinline__ void sk_sum(const double* __restrict__ part, const SkGeom& g,
                                       int64_t c, double& s0, double& s1, double& s2) {
  const int64_t cb = c / kColsPerBlock;
  const int64_t cc = c - cb * kColsPerBlock;
  const int64_t g_lo = sk_owner(g, cb * g.rows);
  const int64_t g_hi = sk_owner(g, (cb + 1) * g.rows - 1);
  s0 = s1 = s2 = 0.0;
  for (int64_t cta = g_lo; cta <= g_hi; ++cta) {
    // fewer units than CTAs (a truncated stream): skip empty ranges
    if (sk_begin(g, cta) == sk_begin(g, cta + 1)) continue;
    const int64_t k = cb - sk_begin(g, cta) / g.rows;
    const double* p = part + ((cta * g.kmax + k) * 3) * kColsPerBlock + cc;
    s0 += p[0];
    s1 += p[kColsPerBlock];
    s2 += p[2 * kColsPerBlock];
  }
}

// kSkLanes lanes cooperate on one column (lane l takes CTAs g_lo+l, +2l, …);
// a fixed xor tree combines them — deterministic, kSkLanes× the MLP.
constexpr int kSkLanes = 4;
__device__ __forceinline__ void sk_sum_lanes(const double* __restrict__ part, const SkGeom& g,
                                             int64_t c, int lane, double& s0, double& s1,
                                             double& s2, bool need = true) {
  const int64_t cb = c / kColsPerBlock;
  const int64_t cc = c - cb * kColsPerBlock;
  const int64_t g_lo = sk_owner(g, cb * g.rows);
  const int64_t g_hi = need ? sk_owner(g, (cb + 1) * g.rows - 1) : g_lo - 1;  // !need: no loads
  s0 = s1 = s2 = 0.0;
  for (int64_t cta = g_lo + lane; cta <= g_hi; cta += kSkLanes) {
    if (sk_begin(g, cta) == sk_begin(g, cta + 1)) continue;  // empty range
    const int64_t k = cb - sk_begin(g, cta) / g.rows;
    const double* p = part + ((cta * g.kmax + k) * 3) * kColsPerBlock + cc;
    s0 += p[0];
    s1 += p[kColsPerBlock];
    s2 += p[2 * kColsPerBlock];
  }
#pragma unroll
  for (int o = kSkLanes / 2; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
}

// A whole warp on one column (lanes stride the covering CTAs, then a fixed
// xor tree): for columns covered by many CTAs (a truncated stream puts the
// whole grid on one column block).
__device__ __forceinline__ void sk_sum_warp(const double* __restrict__ part, const SkGeom& g,
                                            int64_t c, int lane, double& s0, double& s1,
                                            double& s2) {
  const int64_t cb = c / kColsPerBlock;
  const int64_t cc = c - cb * kColsPerBlock;
  const int64_t g_lo = sk_owner(g, cb * g.rows);
  const int64_t g_hi = sk_owner(g, (cb + 1) * g.rows - 1);
  s0 = s1 = s2 = 0.0;
  for (int64_t cta = g_lo + lane; cta <= g_hi; cta += 32) {
    if (sk_begin(g, cta) == sk_begin(g, cta + 1)) continue;
    const int64_t k = cb - sk_begin(g, cta) / g.rows;
    const double* p = part + ((cta * g.kmax + k) * 3) * kColsPerBlock + cc;
    s0 += p[0];
    s1 += p[kColsPerBlock];
    s2 += p[2 * kColsPerBlock];
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
}

SkGeom geom(const ColsumPlan& p) {
  return SkGeom{p.rows, p.cols4, p.units, p.grid, p.kmax, p.trunc};
}
}  // namespace

__global__ void __launch_bounds__(kColsumThreads)
    colsum_kernel(const float* __restrict__ A, int64_t lda, const float4* __restrict__ v,
                  SkGeom g, double* __restrict__ part, const IterState* __restrict__ st,
                  uint64_t* stamps, int stamp_slot) {
  griddep_wait();
  if (st && !st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0)
    stamps[4 * st->iter + stamp_slot] = globaltimer();
  g = sk_eff(g, st);
  const int64_t ld4 = lda >> 2;
  int64_t u = sk_begin(g, blockIdx.x);
  const int64_t u_end = sk_begin(g, blockIdx.x + 1);
  int slot = 0;
  while (u < u_end) {
    const int64_t cb = u / g.rows;
    const int64_t r0 = u - cb * g.rows;
    const int64_t r1 = min(g.rows, r0 + (u_end - u));
    const int64_t c4 = cb * kColsumThreads + threadIdx.x;
    double acc[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;
    if (c4 < g.cols4) {
      const float4* a = reinterpret_cast<const float4*>(A) + c4;
      int64_t r = r0;
      for (; r + kRowGroup <= r1; r += kRowGroup) {
        float4 q[kRowGroup];
#pragma unroll
        for (int w = 0; w < kRowGroup; ++w) q[w] = __ldcs(a + (r + w) * ld4);
        float f[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i][0] = f[i][1] = f[i][2] = 0.f;
#pragma unroll
        for (int w = 0; w < kRowGroup; ++w) {
          const float4 vv = __ldg(v + r + w);
          const float qq[4] = {q[w].x, q[w].y, q[w].z, q[w].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            f[i][0] = __fmaf_rn(qq[i], vv.x, f[i][0]);
            f[i][1] = __fmaf_rn(qq[i], vv.y, f[i][1]);
            f[i][2] = __fmaf_rn(qq[i], vv.z, f[i][2]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i][0] += f[i][0];
          acc[i][1] += f[i][1];
          acc[i][2] += f[i][2];
        }
      }
      for (; r < r1; ++r) {
        const float4 qv = __ldcs(a + r * ld4);
        const float4 vv = __ldg(v + r);
        const float qq[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i][0] += static_cast<double>(qq[i] * vv.x);
          acc[i][1] += static_cast<double>(qq[i] * vv.y);
          acc[i][2] += static_cast<double>(qq[i] * vv.z);
        }
      }
    }
    double* out = part + ((static_cast<int64_t>(blockIdx.x) * g.kmax + slot) * 3) * kColsPerBlock +
                  4 * threadIdx.x;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double2* o = reinterpret_cast<double2*>(out + d * kColsPerBlock);
      o[0] = make_double2(acc[0][d], acc[1][d]);
      o[1] = make_double2(acc[2][d], acc[3][d]);
    }
    u += r1 - r0;
    ++slot;
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) variant: one CTA per SM, a producer warp streams the
// CTA's stream-K row segments into a 6-stage shared-memory ring with
// cp.async.bulk (+ L2 evict-first) completing on mbarriers; 8 consumer warps
// read the stage (conflict-free LDS.128) and accumulate.  Up to 192 KB of
// the basis is in flight per SM regardless of register pressure — the
// long-scoreboard stall that capped the LDG kernel at ~85 % of HBM.
namespace {
constexpr int kBulkStages = 3;       // × 2 CTAs per SM → 192 KB in flight per SM
constexpr int kBulkCtasPerSm = 2;
constexpr int kStageBytes = 32 * 1024;
constexpr int kBulkConsumers = kColsumThreads;         // 8 warps
constexpr int kBulkThreads = kBulkConsumers + 32;      // + producer warp
constexpr int kBulkMaxChunkRows = 64;
constexpr int kBulkVBytes = kBulkMaxChunkRows * 16;   // the chunk's v rows (float4)
constexpr int kBulkSmem = kBulkStages * (kStageBytes + kBulkVBytes) + 2 * kBulkStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// The chunk sequence both roles walk: segments (cb, rows r0..r1) of the
// CTA's stream-K range, each cut into chunks of ≤ chunk_rows rows.
struct SegCursor {
  int64_t u, u_end, cb, r, r1;
  __device__ bool next_segment(const SkGeom& g) {
    if (u >= u_end) return false;
    cb = u / g.rows;
    r = u - cb * g.rows;
    r1 = min(g.rows, r + (u_end - u));
    u += r1 - r;
    return true;
  }
};
}  // namespace

__global__ void __launch_bounds__(kBulkThreads, kBulkCtasPerSm)
    colsum_bulk_kernel(const float* __restrict__ A, int64_t lda, const float4* __restrict__ v,
                       SkGeom g, double* __restrict__ part, const IterState* __restrict__ st,
                       uint64_t* stamps, int stamp_slot) {
  griddep_wait();
  if (st && !st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0)
    stamps[4 * st->iter + stamp_slot] = globaltimer();
  g = sk_eff(g, st);
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);
  float4* vring = reinterpret_cast<float4*>(smem + kBulkStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBulkStages * (kStageBytes + kBulkVBytes));
  uint64_t* empty = full + kBulkStages;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBulkConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = sk_begin(g, blockIdx.x), u1 = sk_begin(g, blockIdx.x + 1);
  const int64_t col_blocks = (g.cols4 + kColsumThreads - 1) / kColsumThreads;

  if (tid >= kBulkConsumers) {  // ---------------- producer warp
    if (tid != kBulkConsumers) return;
    uint64_t policy, policy_v;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy_v));
    SegCursor c{u0, u1, 0, 0, 0};
    int64_t chunk = 0;
    while (c.next_segment(g)) {
      const int64_t c4 = min(static_cast<int64_t>(kColsumThreads), g.cols4 - c.cb * kColsumThreads);
      const uint32_t seg_bytes = static_cast<uint32_t>(c4 * 16);
      const int rows_per_chunk = static_cast<int>(min64(kBulkMaxChunkRows, kStageBytes / seg_bytes));
      const bool contiguous = col_blocks == 1 && lda == 4 * g.cols4;
      for (int64_t r = c.r; r < c.r1; r += rows_per_chunk, ++chunk) {
        const int nr = static_cast<int>(min64(rows_per_chunk, c.r1 - r));
        const int s = static_cast<int>(chunk % kBulkStages);
        const uint32_t ph = static_cast<uint32_t>((chunk / kBulkStages) & 1);
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], seg_bytes * nr + 16u * nr);
        // the chunk's v rows ride along (a broadcast LDG per row stalled the
        // consumers on an L2 round trip)
        bulk_g2s(vring + s * kBulkMaxChunkRows, v + r, 16u * nr, &full[s], policy_v);
        float* dst = ring + static_cast<int64_t>(s) * (kStageBytes / 4);
        const float* src = A + r * lda + c.cb * (4 * kColsumThreads);
        if (contiguous) {
          bulk_g2s(dst, src, seg_bytes * nr, &full[s], policy);
        } else {
          for (int i = 0; i < nr; ++i)
            bulk_g2s(dst + i * (seg_bytes / 4), src + i * lda, seg_bytes, &full[s], policy);
        }
      }
    }
    return;
  }

  // ------------------------------------------------ consumer warps
  SegCursor c{u0, u1, 0, 0, 0};
  int64_t chunk = 0;
  int slot = 0;
  while (c.next_segment(g)) {
    const int64_t c4 = min(static_cast<int64_t>(kColsumThreads), g.cols4 - c.cb * kColsumThreads);
    const uint32_t seg_bytes = static_cast<uint32_t>(c4 * 16);
    const int rows_per_chunk = static_cast<int>(min64(kBulkMaxChunkRows, kStageBytes / seg_bytes));
    const bool active = tid < c4;
    double acc[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;
    for (int64_t r = c.r; r < c.r1; r += rows_per_chunk, ++chunk) {
      const int nr = static_cast<int>(min64(rows_per_chunk, c.r1 - r));
      const int s = static_cast<int>(chunk % kBulkStages);
      const uint32_t ph = static_cast<uint32_t>((chunk / kBulkStages) & 1);
      mbar_wait(&full[s], ph);
      if (active) {
        const float4* row = reinterpret_cast<const float4*>(ring + static_cast<int64_t>(s) * (kStageBytes / 4)) + tid;
        const int stride4 = static_cast<int>(seg_bytes / 16);
        float f[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i][0] = f[i][1] = f[i][2] = 0.f;
        auto fma_row = [&](const float4 q, const float4 vv) {
          const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            f[j][0] = __fmaf_rn(qq[j], vv.x, f[j][0]);
            f[j][1] = __fmaf_rn(qq[j], vv.y, f[j][1]);
            f[j][2] = __fmaf_rn(qq[j], vv.z, f[j][2]);
          }
        };
        auto flush = [&] {  // fp32 over ≤ 8 rows, then fp64
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[j][0] += f[j][0];
            acc[j][1] += f[j][1];
            acc[j][2] += f[j][2];
            f[j][0] = f[j][1] = f[j][2] = 0.f;
          }
        };
        const float4* vs = vring + s * kBulkMaxChunkRows;
        int i = 0;
        for (; i + 8 <= nr; i += 8) {  // 8 independent LDS + 8 broadcast LDS
          float4 vv[8], q[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) vv[w] = vs[i + w];
#pragma unroll
          for (int w = 0; w < 8; ++w) q[w] = row[(i + w) * stride4];
#pragma unroll
          for (int w = 0; w < 8; ++w) fma_row(q[w], vv[w]);
          flush();
        }
        for (; i < nr; ++i) fma_row(row[i * stride4], vs[i]);
        flush();
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    double* out = part + ((static_cast<int64_t>(blockIdx.x) * g.kmax + slot) * 3) * kColsPerBlock +
                  4 * tid;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double2* o = reinterpret_cast<double2*>(out + d * kColsPerBlock);
      o[0] = make_double2(acc[0][d], acc[1][d]);
      o[1] = make_double2(acc[2][d], acc[3][d]);
    }
    ++slot;
  }
}

// ---------------------------------------------------------------------------
// z = Qᵀ·R as ROW dot products over Qᵀ (K × M row-major fp32).  With
// spectral truncation the streamed eigenvectors are a contiguous PREFIX of
// Qᵀ's rows, so every copy is a long contiguous run; over Q (M × K
// row-major) the same prefix is a short strided piece of every row (C4:
// 736 of 1200 bytes per row, 2.3 TB/s).  Work units are (group of
// kRdRows eigenvector rows, 1024-column block); a persistent stream-K grid
// splits them evenly in row-group-major order.  A producer warp bulk-copies
// a unit's kRdRows × 4 KB row pieces (L2 evict-first) and its 16 KB of R
// into a stage of a 4-stage ring; 8 consumer warps: each thread owns 4
// columns, reads their R from the stage and keeps
// kRdRows × 3 sums for the current row group (fp32 over the unit's 4
// products per column thread, then fp64).  When the CTA leaves a row group it reduces its threads in a
// fixed order into one partial slot; rowdot_reduce sums a row's slots in
// CTA order — bitwise reproducible.
namespace {
constexpr int kRdRows = 8;                        // eigenvector rows per unit
constexpr int kRdCols = 4 * kColsumThreads;       // 1024 columns per unit
// columns per consumer thread (2, with 16 consumer warps: 46 µs against 44
// at C4 — register-capped with spills)
constexpr int kRdCpt = 4;
constexpr int kRdConsumers = kRdCols / kRdCpt;    // consumer threads
constexpr int kRdThreads = kRdConsumers + 32;     // + producer warp
constexpr int kRdSlot = kRdRows * 3;              // doubles per partial slot
// one CTA per SM with a 4-stage ring of (32 KB of Qᵀ + the unit's 16 KB of
// R): the 8×3 fp64 sums per thread need the registers of a single resident
// CTA; 128 KB of the basis in flight per SM
constexpr int kRdStages = 4;
constexpr int kRdRBytes = kRdCols * 16;           // the unit's R columns (float4)
constexpr int kRdSmem = kRdStages * (kStageBytes + kRdRBytes) + 2 * kRdStages * 8;

__device__ __forceinline__ RdGeom rd_eff(RdGeom g, const IterState* st) {
  if (!g.trunc || !st) return g;
  g.rows = min(g.rows, static_cast<int64_t>(st->keff));
  g.units = (g.rows + kRdRows - 1) / kRdRows * g.col_blocks;
  return g;
}
__host__ __device__ __forceinline__ int64_t rd_begin(const RdGeom& g, int64_t cta) {
  return cta * g.units / g.grid;
}
__device__ __forceinline__ int64_t rd_owner(const RdGeom& g, int64_t u) {
  return ((u + 1) * g.grid - 1) / g.units;
}
}  // namespace

__global__ void __launch_bounds__(kRdThreads, 1)
    rowdot_bulk_kernel(const float* __restrict__ A, const float4* __restrict__ v, RdGeom g,
                       double* __restrict__ part, const IterState* __restrict__ st,
                       uint64_t* stamps, int stamp_slot) {
  griddep_wait();
  if (st && !st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0)
    stamps[4 * st->iter + stamp_slot] = globaltimer();
  g = rd_eff(g, st);
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);
  float4* rring = reinterpret_cast<float4*>(smem + kRdStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRdStages * (kStageBytes + kRdRBytes));
  uint64_t* empty = full + kRdStages;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kRdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRdConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = rd_begin(g, blockIdx.x), u1 = rd_begin(g, blockIdx.x + 1);
  static_assert(kRdRows * kRdCols * 4 == kStageBytes, "one unit per stage");

  if (tid >= kRdConsumers) {  // ---------------- producer warp
    if (tid != kRdConsumers) return;
    uint64_t policy, policy_r;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy_r));
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t chunk = u - u0;
      const int s = static_cast<int>(chunk % kRdStages);
      const uint32_t ph = static_cast<uint32_t>((chunk / kRdStages) & 1);
      const int64_t rg = u / g.col_blocks, cb = u - rg * g.col_blocks;
      const int64_t c0 = cb * kRdCols;
      const int64_t ncol = min(static_cast<int64_t>(kRdCols), g.cols - c0);
      const uint32_t bytes = static_cast<uint32_t>(((ncol + 3) & ~int64_t(3)) * 4);
      const int nrows = static_cast<int>(min(static_cast<int64_t>(kRdRows), g.rows - rg * kRdRows));
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t rbytes = static_cast<uint32_t>(ncol * 16);
      mbar_expect_tx(&full[s], bytes * nrows + rbytes);
      bulk_g2s(rring + s * kRdCols, v + c0, rbytes, &full[s], policy_r);  // R of the unit
      float* dst = ring + static_cast<int64_t>(s) * (kStageBytes / 4);
      for (int r = 0; r < nrows; ++r)
        bulk_g2s(dst + r * kRdCols, A + (rg * kRdRows + r) * g.lda + c0, bytes, &full[s], policy);
    }
    return;
  }

  // ------------------------------------------------ consumer warps
  __shared__ double red[kRdConsumers / 32][kRdSlot];
  // per row and unit: an fp32 dot product over the thread's kRdCpt columns,
  // then fp64 (fp32 over several units: 1e-6 worse σ² agreement with the
  // fused path at C0, no speed-up)
  double acc[kRdRows][3];
#pragma unroll
  for (int r = 0; r < kRdRows; ++r) acc[r][0] = acc[r][1] = acc[r][2] = 0.0;
  int slot = 0;
  // the fixed-order CTA reduction of the current row group into slot `slot`
  auto flush_group = [&]() {
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int r = 0; r < kRdRows; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = warp_sum(acc[r][c]);
        if (lane == 0) red[warp][r * 3 + c] = w;
        acc[r][c] = 0.0;
      }
    asm volatile("bar.sync 1, %0;" ::"r"(kRdConsumers));  // consumers only
    if (tid < kRdSlot) {
      double s = 0.0;
      for (int w = 0; w < kRdConsumers / 32; ++w) s += red[w][tid];
      part[(static_cast<int64_t>(blockIdx.x) * g.kmax + slot) * kRdSlot + tid] = s;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kRdConsumers));  // red is reused
    ++slot;
  };
  int64_t cur_rg = u0 < u1 ? u0 / g.col_blocks : 0;
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t chunk = u - u0;
    const int s = static_cast<int>(chunk % kRdStages);
    const uint32_t ph = static_cast<uint32_t>((chunk / kRdStages) & 1);
    const int64_t rg = u / g.col_blocks, cb = u - rg * g.col_blocks;
    if (rg != cur_rg) {
      flush_group();
      cur_rg = rg;
    }
    const int64_t c0 = cb * kRdCols + kRdCpt * tid;
    const int nrows = static_cast<int>(min(static_cast<int64_t>(kRdRows), g.rows - rg * kRdRows));
    mbar_wait(&full[s], ph);
    // R of the thread's kRdCpt columns, staged with the unit (a per-unit L2
    // round trip otherwise serialises the consumers)
    float4 rv[kRdCpt];
    const float4* rs = rring + s * kRdCols + kRdCpt * tid;
#pragma unroll
    for (int j = 0; j < kRdCpt; ++j)
      rv[j] = c0 + j < g.cols ? rs[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float* stf = ring + static_cast<int64_t>(s) * (kStageBytes / 4);
#pragma unroll
    for (int r = 0; r < kRdRows; ++r) {
      if (r < nrows && c0 < g.cols) {
        // fp32 over the thread's kRdCpt columns, then fp64
        static_assert(kRdCpt == 4, "one float4 of the basis row per thread");
        const float4 q4 = reinterpret_cast<const float4*>(stf)[r * (kRdCols / 4) + tid];
        const float q[kRdCpt] = {q4.x, q4.y, q4.z, q4.w};
        float fx = q[0] * rv[0].x, fy = q[0] * rv[0].y, fz = q[0] * rv[0].z;
#pragma unroll
        for (int j = 1; j < kRdCpt; ++j) {
          fx = __fmaf_rn(q[j], rv[j].x, fx);
          fy = __fmaf_rn(q[j], rv[j].y, fy);
          fz = __fmaf_rn(q[j], rv[j].z, fz);
        }
        acc[r][0] += static_cast<double>(fx);
        acc[r][1] += static_cast<double>(fy);
        acc[r][2] += static_cast<double>(fz);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (u0 < u1) flush_group();
}

// z_k (k < rows this iteration) = Σ over the CTAs covering its row group of
// their slot, in CTA order (a warp per k: lanes stride the CTAs, fixed xor
// tree).  filter != 0: c = z/(λ + λ_reg σ²), g = λnum·c (zreduce_filter);
// else z (SoA 3×K, zeros past the streamed rows) for the distributed
// all-reduce.
__global__ void rowdot_reduce_kernel(const double* __restrict__ part, RdGeom g, int64_t k,
                                     const double* __restrict__ lam,
                                     const double* __restrict__ lam_num, double lambda_reg,
                                     double* __restrict__ coef, float4* __restrict__ g4,
                                     double* __restrict__ z_out, IterState* st) {
  griddep_wait();
  if (st && !st->active) return;
  g = rd_eff(g, st);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t kk = min(k, g.rows);
  const double sigma2 = st ? st->sigma2 : 0.0;
  if (st && lam && warp == 0 && lane == 0) st->sigma2_m = sigma2;
  for (int64_t i = warp; i < (z_out ? k : kk); i += nwarps) {
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    if (i < kk) {
      const int64_t rg = i / kRdRows, rr = i - rg * kRdRows;
      const int64_t g0 = rd_owner(g, rg * g.col_blocks), g1 = rd_owner(g, (rg + 1) * g.col_blocks - 1);
      for (int64_t cta = g0 + lane; cta <= g1; cta += 32) {
        const int64_t b = rd_begin(g, cta);
        if (b == rd_begin(g, cta + 1)) continue;  // empty range
        const int64_t slot = rg - b / g.col_blocks;
        const double* p = part + (cta * g.kmax + slot) * kRdSlot + rr * 3;
        z0 += p[0];
        z1 += p[1];
        z2 += p[2];
      }
      z0 = warp_sum(z0);
      z1 = warp_sum(z1);
      z2 = warp_sum(z2);
    }
    if (lane) continue;
    if (z_out) {
      z_out[i] = z0;
      z_out[k + i] = z1;
      z_out[2 * k + i] = z2;
      continue;
    }
    const double diag = lam[i] + lambda_reg * sigma2;
    if (!(diag > 0.0)) set_error(st, kDevSolveDiag, diag);
    const double inv = 1.0 / diag;
    coef[i] = z0 * inv;
    coef[k + i] = z1 * inv;
    coef[2 * k + i] = z2 * inv;
    const double f = lam_num[i] * inv;
    g4[i] = make_float4(static_cast<float>(z0 * f), static_cast<float>(z1 * f),
                        static_cast<float>(z2 * f), 0.f);
  }
}

RowdotPlan make_rowdot_plan(int64_t k, int64_t m, int64_t lda, int sm_count) {
  RowdotPlan p;
  p.g.rows = k;
  p.g.cols = m;
  p.g.lda = lda;
  p.g.col_blocks = (m + kRdCols - 1) / kRdCols;
  p.g.units = (k + kRdRows - 1) / kRdRows * p.g.col_blocks;
  static bool attr = false;
  if (!attr) {
    FCPD_CUDA(cudaFuncSetAttribute(rowdot_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kRdSmem));
    attr = true;
  }
  p.g.grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(static_cast<int64_t>(sm_count), p.g.units)));
  // slots per CTA: the row groups its range can touch (+1: a truncated
  // geometry may cross one more boundary)
  const int64_t per = (p.g.units + p.g.grid - 1) / p.g.grid;
  p.g.kmax = static_cast<int>((per + p.g.col_blocks - 1) / p.g.col_blocks + 2);
  return p;
}

size_t RowdotPlan::part_doubles() const {
  return static_cast<size_t>(g.grid) * g.kmax * kRdSlot;
}

void launch_rowdot(const RowdotPlan& p, const float* qt, const float4* v, double* part,
                   const IterState* st, uint64_t* stamps, int stamp_slot, cudaStream_t stream) {
  launch_pdl(rowdot_bulk_kernel, dim3(p.g.grid), dim3(kRdThreads), kRdSmem, stream, qt, v,
             p.g, part, st, stamps, stamp_slot);
  FCPD_LAUNCH_CHECK();
}

void launch_rowdot_reduce(const RowdotPlan& p, const double* part, int64_t k, const double* lam,
                          const double* lam_num, double lambda_reg, double* coef, float4* g4,
                          double* z_out, IterState* st, cudaStream_t stream) {
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(k * 32, 256), 148 * 2));
  launch_pdl(rowdot_reduce_kernel, dim3(blocks), dim3(256), 0, stream, part, p.g, k, lam,
             lam_num, lambda_reg, coef, g4, z_out, st);
  FCPD_LAUNCH_CHECK();
}

// z_k = Σ partials; solve + filter (solvers.hpp:66-72):
//   c_k = z_k / (λ_k + λ_reg σ²)   (W = Q c, kept for `coefficients`)
//   g_k = λnum_k · c_k             (ΦW = Q g)
__global__ void zreduce_filter_kernel(const double* __restrict__ part, SkGeom g, int64_t k,
                                      const double* __restrict__ lam,
                                      const double* __restrict__ lam_num, double lambda_reg,
                                      double* __restrict__ coef, float4* __restrict__ g4,
                                      IterState* st) {
  griddep_wait();
  if (!st->active) return;
  g = sk_eff(g, st);
  // one warp per column, grid-stride over the K columns
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t kk = g.trunc == 1 ? min(k, g.cols4 * 4) : k;  // streamed eigenvectors
  // σ² of this iteration's E-step, unclamped (registration.hpp:137)
  const double sigma2 = st->sigma2;
  if (warp == 0 && lane == 0) st->sigma2_m = sigma2;
  // columns ≥ kk (filter below tau) are neither streamed nor read this
  // iteration: V stops at the same keff, and the final coefficients are
  // recomputed over the full basis (launch_zcoef)
  for (int64_t i = warp; i < kk; i += nwarps) {
    double z0, z1, z2;
    sk_sum_warp(part, g, i, lane, z0, z1, z2);
    if (lane) continue;
    const double diag = lam[i] + lambda_reg * sigma2;
    if (!(diag > 0.0)) set_error(st, kDevSolveDiag, diag);
    const double inv = 1.0 / diag;
    coef[i] = z0 * inv;
    coef[k + i] = z1 * inv;
    coef[2 * k + i] = z2 * inv;
    const double f = lam_num[i] * inv;
    g4[i] = make_float4(static_cast<float>(z0 * f), static_cast<float>(z1 * f),
                        static_cast<float>(z2 * f), 0.f);
  }
}

// x̃new = X + V; per-row σ² terms; block partial sums (fixed order).
__global__ void __launch_bounds__(256)
    transform_sigma_kernel(const double* __restrict__ part, SkGeom g, int64_t m,
                           int64_t m_valid, const double* __restrict__ x0, double* xt64,
                           double* __restrict__ xt_prev, float4* __restrict__ xt4,
                           const double* __restrict__ ptilde_y, const double* __restrict__ var,
                           double* __restrict__ sig_part, IterState* st, uint64_t* stamps) {
  griddep_wait();
  // m = row stride of the SoA arrays; rows ≥ m_valid (shard padding) are inert
  if (!st->active) return;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0) stamps[4 * st->iter + 2] = globaltimer();
  g = sk_eff(g, st);
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = gid / kSkLanes;
  double term = 0.0;
  double v0, v1, v2;
  sk_sum_lanes(part, g, i < m ? i : m - 1, static_cast<int>(gid % kSkLanes), v0, v1, v2);
  if (i < m_valid && gid % kSkLanes == 0) {
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
  griddep_wait();
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
  finish_iteration_sigma(st, tot, m, d, early_stop, trace, stamps);
}

// out = X + Σ partials  (apply_transform_lowrank epilogue, no σ² terms)
__global__ void vreduce_add_kernel(const double* __restrict__ part, SkGeom g, int64_t m,
                                   const double* __restrict__ x0, int d,
                                   double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double v[3];
  sk_sum(part, g, i, v[0], v[1], v[2]);
  for (int c = 0; c < d; ++c) out[c * m + i] = (x0 ? x0[c * m + i] : 0.0) + v[c];
}

// Effective spectral rank: f_k = λnum_k/(λ_k + λ_reg σ²) is non-increasing
// along the descending spectrum (λnum = λ_raw or λ, both sorted), so the
// kept eigenpairs are a prefix: cta_spectral_rank (mstep.cuh) finds the
// first f_k < tau.
// Dropping them changes V = Q(f ⊙ z) by ≤ Σ_{dropped} f_k |z_k| |q_k| —
// with tau = 1e-10 far below the fp32 basis rounding (≈ 2e-7‖R‖).
__global__ void spectral_rank_kernel(const double* __restrict__ lam,
                                     const double* __restrict__ lam_num, int64_t k,
                                     double lambda_reg, double tau, IterState* st) {
  griddep_wait();
  if (!st->active) return;
  int64_t keep = k;
  if (tau > 0.0) keep = cta_spectral_rank(lam, lam_num, k, lambda_reg * st->sigma2, tau);
  if (threadIdx.x != 0) return;
  keep = (keep + 3) / 4 * 4;
  st->keff = static_cast<int32_t>(min(max(keep, int64_t(4)), (k + 3) / 4 * 4));
}

__global__ void zcoef_kernel(const double* __restrict__ part, SkGeom g, int64_t k,
                             const double* __restrict__ lam, double lambda_reg,
                             double* __restrict__ coef, const IterState* __restrict__ st) {
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = gid / kSkLanes;
  double z0, z1, z2;
  sk_sum_lanes(part, g, i < k ? i : k - 1, static_cast<int>(gid % kSkLanes), z0, z1, z2);
  if (i >= k || gid % kSkLanes) return;
  const double inv = 1.0 / (lam[i] + lambda_reg * st->sigma2_m);
  coef[i] = z0 * inv;
  coef[k + i] = z1 * inv;
  coef[2 * k + i] = z2 * inv;
}

void launch_spectral_rank(const double* lam, const double* lam_num, int64_t k, double lambda_reg,
                          double tau, IterState* st, cudaStream_t stream) {
  launch_pdl(spectral_rank_kernel, dim3(1), dim3(512), 0, stream, lam, lam_num, k, lambda_reg, tau,
             st);
  FCPD_LAUNCH_CHECK();
}

void launch_zcoef(const ColsumPlan& p, const double* part, const double* lam, double lambda_reg,
                  double* coef, const IterState* st, cudaStream_t stream) {
  SkGeom g = geom(p);
  g.trunc = 0;
  zcoef_kernel<<<ceil_div(p.cols * kSkLanes, 256), 256, 0, stream>>>(part, g, p.cols, lam,
                                                                     lambda_reg, coef, st);
  FCPD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------

ColsumPlan make_colsum_plan(int64_t rows, int64_t cols, int sm_count, int ctas_per_sm) {
  ColsumPlan p;
  p.rows = rows;
  p.cols = cols;
  p.cols4 = (cols + 3) / 4;
  p.col_blocks = ceil_div(p.cols4, kColsumThreads);
  p.units = p.rows * p.col_blocks;
  // FCPD_COLSUM=ldg selects the register-staged LDG kernel (A/B measurement)
  const char* env = std::getenv("FCPD_COLSUM");
  p.bulk = !(env && std::string(env) == "ldg");
  int64_t slots = 0;
  if (p.bulk) {
    static bool attr = false;
    if (!attr) {
      FCPD_CUDA(cudaFuncSetAttribute(colsum_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBulkSmem));
      attr = true;
    }
    slots = static_cast<int64_t>(sm_count) * std::max(1, std::min(ctas_per_sm, kBulkCtasPerSm));
  } else {
    int occ = 0;
    FCPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, colsum_kernel, kColsumThreads, 0));
    slots = static_cast<int64_t>(sm_count) * std::max(occ, 1);
  }
  p.grid = static_cast<int>(std::max<int64_t>(1, min64(slots, p.units)));
  const int64_t per = (p.units + p.grid - 1) / p.grid;
  // + 1: a truncated geometry (sk_eff) may cross one more block boundary
  p.kmax = static_cast<int>((per + rows - 1) / rows + 2);
  return p;
}

void launch_colsum(const ColsumPlan& p, const float* A, int64_t lda, const float4* v,
                   double* part, const IterState* st, uint64_t* stamps, int stamp_slot,
                   cudaStream_t stream) {
  if (p.bulk)
    launch_pdl(colsum_bulk_kernel, dim3(p.grid), dim3(kBulkThreads), kBulkSmem, stream, A, lda, v,
               geom(p), part, st, stamps, stamp_slot);
  else
    launch_pdl(colsum_kernel, dim3(p.grid), dim3(kColsumThreads), 0, stream, A, lda, v, geom(p),
               part, st, stamps, stamp_slot);
  FCPD_LAUNCH_CHECK();
}

void launch_zreduce(const ColsumPlan& p, const double* part, const double* lam,
                    const double* lam_num, double lambda_reg, double* coef, float4* g4,
                    IterState* st, cudaStream_t stream) {
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(p.cols * 32, 256), 148 * 2));
  launch_pdl(zreduce_filter_kernel, dim3(blocks), dim3(256), 0, stream, part, geom(p), p.cols, lam,
             lam_num, lambda_reg, coef, g4, st);
  FCPD_LAUNCH_CHECK();
}

void launch_transform_sigma(const ColsumPlan& p, const double* part, const double* x0,
                            double* xt64, double* xt_prev, float4* xt4,
                            const double* ptilde_y, const double* var, double* sig_part,
                            int d, int early_stop, double* trace, IterState* st,
                            uint64_t* stamps, cudaStream_t stream) {
  const int64_t m = p.cols;
  const int nb = launch_transform_rows(p, part, m, x0, xt64, xt_prev, xt4, ptilde_y, var,
                                       sig_part, st, stamps, stream);
  launch_sigma_final(sig_part, nb, m, d, early_stop, trace, st, stamps, stream);
}

int transform_sigma_blocks(int64_t m) { return ceil_div(m * kSkLanes, 256); }

int launch_transform_rows(const ColsumPlan& p, const double* part, int64_t m_valid,
                          const double* x0, double* xt64, double* xt_prev, float4* xt4,
                          const double* ptilde_y, const double* var, double* sig_part,
                          IterState* st, uint64_t* stamps, cudaStream_t stream) {
  const int64_t m = p.cols;
  const int nb = transform_sigma_blocks(m);
  launch_pdl(transform_sigma_kernel, dim3(nb), dim3(256), 0, stream, part, geom(p), m, m_valid, x0,
             xt64, xt_prev, xt4, ptilde_y, var, sig_part, st, stamps);
  FCPD_LAUNCH_CHECK();
  return nb;
}

void launch_sigma_final(const double* sig_part, int blocks, int64_t m_global, int d,
                        int early_stop, double* trace, IterState* st, uint64_t* stamps,
                        cudaStream_t stream) {
  launch_pdl(sigma_final_kernel, dim3(1), dim3(256), 0, stream, sig_part, blocks, m_global, d,
             early_stop, trace, st, stamps);
  FCPD_LAUNCH_CHECK();
}

// z (SoA 3×K) = Σ stream-K partials, no filter (distributed path: all-reduced
// next).  One warp per column; columns outside this iteration's truncated
// stream are zero so the all-reduce carries no stale values.
__global__ void zsum_kernel(const double* __restrict__ part, SkGeom g, int64_t k,
                            double* __restrict__ z, const IterState* __restrict__ st) {
  if (st && !st->active) return;
  g = sk_eff(g, st);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t kk = g.trunc == 1 ? min(k, g.cols4 * 4) : k;
  for (int64_t i = warp; i < k; i += nwarps) {
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    if (i < kk) sk_sum_warp(part, g, i, lane, z0, z1, z2);
    if (lane) continue;
    z[i] = z0;
    z[k + i] = z1;
    z[2 * k + i] = z2;
  }
}

__global__ void zfilter_kernel(const double* __restrict__ z, int64_t k,
                               const double* __restrict__ lam, const double* __restrict__ lam_num,
                               double lambda_reg, double* __restrict__ coef,
                               float4* __restrict__ g4, IterState* st) {
  if (!st->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  if (i == 0) st->sigma2_m = st->sigma2;
  const double diag = lam[i] + lambda_reg * st->sigma2;
  if (!(diag > 0.0)) set_error(st, kDevSolveDiag, diag);
  const double inv = 1.0 / diag;
  const double z0 = z[i], z1 = z[k + i], z2 = z[2 * k + i];
  coef[i] = z0 * inv;
  coef[k + i] = z1 * inv;
  coef[2 * k + i] = z2 * inv;
  const double f = lam_num[i] * inv;
  g4[i] = make_float4(static_cast<float>(z0 * f), static_cast<float>(z1 * f),
                      static_cast<float>(z2 * f), 0.f);
}

void launch_zsum(const ColsumPlan& p, const double* part, double* z, const IterState* st,
                 cudaStream_t stream) {
  SkGeom g = geom(p);
  if (!st) g.trunc = 0;  // host-driven full sum
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(p.cols * 32, 256), 148 * 2));
  zsum_kernel<<<blocks, 256, 0, stream>>>(part, g, p.cols, z, st);
  FCPD_LAUNCH_CHECK();
}

// coef = z / (λ + λ_reg σ²_m) from an assembled z (distributed final coefficients)
__global__ void zcoef_full_kernel(const double* __restrict__ z, int64_t k,
                                  const double* __restrict__ lam, double lambda_reg,
                                  double* __restrict__ coef, const IterState* __restrict__ st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double inv = 1.0 / (lam[i] + lambda_reg * st->sigma2_m);
  coef[i] = z[i] * inv;
  coef[k + i] = z[k + i] * inv;
  coef[2 * k + i] = z[2 * k + i] * inv;
}

void launch_zcoef_full(const double* z, int64_t k, const double* lam, double lambda_reg,
                       double* coef, const IterState* st, cudaStream_t stream) {
  zcoef_full_kernel<<<ceil_div(k, 256), 256, 0, stream>>>(z, k, lam, lambda_reg, coef, st);
  FCPD_LAUNCH_CHECK();
}

void launch_zfilter(const double* z, int64_t k, const double* lam, const double* lam_num,
                    double lambda_reg, double* coef, float4* g4, IterState* st,
                    cudaStream_t stream) {
  zfilter_kernel<<<ceil_div(k, 256), 256, 0, stream>>>(z, k, lam, lam_num, lambda_reg, coef, g4,
                                                       st);
  FCPD_LAUNCH_CHECK();
}

void launch_vreduce_add(const ColsumPlan& p, const double* part, const double* x0, int d,
                        double* out, cudaStream_t stream) {
  SkGeom g = geom(p);
  g.trunc = 0;  // host-driven full products (no IterState)
  vreduce_add_kernel<<<ceil_div(p.cols, 256), 256, 0, stream>>>(part, g, p.cols, x0, d, out);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
