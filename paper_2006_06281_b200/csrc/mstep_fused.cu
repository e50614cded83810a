// mstep_fused.cu — the whole M-step of one iteration (solvers.hpp:61-73,
// :138-155, :160-176) as ONE cooperative persistent kernel, for bases whose
// streamed part stays in L2 (single GPU).
//
// The streaming path (mstep.cu) is two HBM-bound passes over Q and Qᵀ plus
// three small kernels.  When the streamed basis is small — the truncated
// full-rank basis of C1 (keff ≈ 150–200 of 20 000 eigenpairs: 15 MB), the
// K = 200 basis of C2 (40 MB), C0 — those passes are latency-bound and the
// launch chain dominates.  One kernel does all of it with grid-wide syncs:
//   phase 0  keff (spectral truncation; every CTA evaluates the same search)
//   phase 1  z partials: CTA c sums Q[r][k]·R_r over its row slice r ∈ [r0, r1)
//   phase 2  z_k = Σ_c partials (fixed order), c_k = z_k/(λ_k + λ_reg σ²),
//            g_k = λnum_k·c_k                       — one warp per k
//   phase 3  V_r = Σ_k Q[r][k]·g_k for the same row slice (Q rows re-read
//            from L2, not Qᵀ), x̃new = X + V, per-row σ² terms (mstep.cu)
//   phase 4  σ² = Σ terms / (D·M), checks, trace, early stop (the last CTA
//            to finish phase 3; no grid barrier)
// Every sum has a fixed order: bitwise reproducible.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "estep_device.cuh"
#include "mstep.cuh"

namespace cg = cooperative_groups;

namespace fcpd {

// FCPD_SMALL_PROBE (diagnostic builds): CTA 0's globaltimer at the phase
// boundaries of one iteration, printed by the CTA that finishes it
#ifdef FCPD_SMALL_PROBE
__device__ unsigned long long g_probe[10];
#define SMALL_PROBE(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_probe[i] = globaltimer();
#else
#define SMALL_PROBE(i)
#endif

namespace {
constexpr int kFusedThreads = 512;
constexpr int kFusedWarps = kFusedThreads / 32;
// phase 1: 12 doubles per thread; phase 3: 3 floats × S slots × (8·ng + 1)
// padded rows, S·ng ≤ kFusedThreads
constexpr int kFusedSmem = 3 * 9 * kFusedThreads * 4;
static_assert(kFusedSmem >= kFusedThreads * 12 * 8, "phase-1 partials fit");
// Phase 3 reads g (K float4) from shared memory: every CTA reading the same
// few L2 lines directly is a hot spot (measured: +10 µs at C1).
constexpr int kG4Max = 8192;  // 128 KB: every fused-path basis up to K = 8192
constexpr int kFusedDynSmem = kFusedSmem + kG4Max * 16;

// spectral_rank_kernel (mstep.cu), as a parallel CTA search
__device__ __forceinline__ int64_t fused_keff(const MstepFusedArgs& a) {
  int64_t keep = a.k;
  if (a.trunc && a.tau > 0.0)
    keep = cta_spectral_rank(a.lam, a.lam_num, a.k, a.lambda_reg * a.st->sigma2, a.tau);
  keep = (keep + 3) / 4 * 4;
  return min(max(keep, int64_t(4)), (a.k + 3) / 4 * 4);
}
}  // namespace

// The fused M-step for the CTA's grid (a cooperative launch of kFusedThreads
// threads with kFusedDynSmem of dynamic shared memory): mstep_fused_kernel,
// and the tail of small_iter_kernel.
__device__ __forceinline__ void mstep_fused_body(const MstepFusedArgs& a) {
  IterState* st = a.st;
  if (!st->active) return;  // uniform: nothing below writes `active` before the last sync
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int it = st->iter;
  if (a.stamps && c == 0 && tid == 0) a.stamps[4 * it + 1] = globaltimer();

  // phases 1 and 3 share the first kFusedSmem bytes; g (phase 3) follows
  extern __shared__ __align__(16) unsigned char fused_smem[];
  // ---- phase 0: effective rank
  const int64_t keff = fused_keff(a);
  if (c == 0 && tid == 0) st->keff = static_cast<int32_t>(keff);
  const int64_t m = a.m;
  const int64_t r0 = c * m / G, r1 = (c + 1) * m / G;
  const int nq = static_cast<int>(keff / 4);  // float4 quads of the streamed columns

  SMALL_PROBE(4);
  // ---- phase 1: z partials over the CTA's rows.  Threads = (row group, quad).
  double* red = reinterpret_cast<double*>(fused_smem);  // [12][thread]
  {
    const int ng = nq >= kFusedThreads ? 1 : kFusedThreads / nq;
    const int grp = nq >= kFusedThreads ? 0 : tid / nq;
    for (int qb = 0; qb < nq; qb += (nq >= kFusedThreads ? kFusedThreads : nq)) {
      const int q = qb + (nq >= kFusedThreads ? tid : tid % nq);
      const bool on = grp < ng && q < nq;
      double acc[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) acc[i] = 0.0;
      if (on) {
        const float4* col = reinterpret_cast<const float4*>(a.q) + q;
        const int64_t ld4 = a.kpad / 4;
        for (int64_t r = r0 + grp; r < r1; r += 8 * ng) {  // 8 rows in flight, fp32 over 8
          float4 qv[8], rv[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const bool in = r + w * ng < r1;  // rows past the slice contribute 0
            qv[w] = in ? __ldg(col + (r + w * ng) * ld4) : make_float4(0.f, 0.f, 0.f, 0.f);
            rv[w] = in ? __ldcg(a.resid4 + r + w * ng) : make_float4(0.f, 0.f, 0.f, 0.f);
          }

          float f[12];
#pragma unroll
          for (int i = 0; i < 12; ++i) f[i] = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const float qq[4] = {qv[w].x, qv[w].y, qv[w].z, qv[w].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              f[3 * i] = __fmaf_rn(qq[i], rv[w].x, f[3 * i]);
              f[3 * i + 1] = __fmaf_rn(qq[i], rv[w].y, f[3 * i + 1]);
              f[3 * i + 2] = __fmaf_rn(qq[i], rv[w].z, f[3 * i + 2]);
            }
          }
#pragma unroll
          for (int i = 0; i < 12; ++i) acc[i] += f[i];
        }
      }
      if (ng > 1) {  // combine the row groups in group order
        __syncthreads();
        if (on)
#pragma unroll
          for (int i = 0; i < 12; ++i) red[i * kFusedThreads + tid] = acc[i];
        __syncthreads();
        if (tid < nq) {
          for (int i = 0; i < 12; ++i) acc[i] = red[i * kFusedThreads + tid];
          for (int gg = 1; gg < ng; ++gg)
#pragma unroll
            for (int i = 0; i < 12; ++i) acc[i] += red[i * kFusedThreads + gg * nq + tid];
        }
      }
      if ((ng > 1 && tid < nq) || (ng == 1 && on)) {
        const int qq = ng > 1 ? tid : q;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // keff is a multiple of 4 and may exceed K (padding columns of Q,
          // all zero): only real eigenpairs have partial slots
          if (4 * qq + i >= a.k) break;
          double* p = a.zpart + ((static_cast<int64_t>(4 * qq + i) * G + c) * 3);
          p[0] = acc[3 * i];
          p[1] = acc[3 * i + 1];
          p[2] = acc[3 * i + 2];
        }
      }
    }
  }
  SMALL_PROBE(5);
  grid.sync();
  SMALL_PROBE(6);

  // ---- phase 2: reduce + solve + filter, one warp per eigenpair
  {
    const double sigma2 = st->sigma2;  // this iteration's E-step σ² (registration.hpp:137)
    const int64_t gw = static_cast<int64_t>(c) * kFusedWarps + warp, nw = int64_t(G) * kFusedWarps;
    for (int64_t k = gw; k < keff; k += nw) {
      if (k >= a.k) {  // padding column of the last quad: g = 0 (Q's column is 0)
        if (lane == 0) a.g4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      double z0 = 0.0, z1 = 0.0, z2 = 0.0;
      for (int cc = lane; cc < G; cc += 32) {
        const double* p = a.zpart + (k * G + cc) * 3;  // written by other CTAs
        z0 += __ldcg(p);
        z1 += __ldcg(p + 1);
        z2 += __ldcg(p + 2);
      }
      z0 = warp_sum(z0);
      z1 = warp_sum(z1);
      z2 = warp_sum(z2);
      if (lane) continue;
      const double diag = a.lam[k] + a.lambda_reg * sigma2;
      if (!(diag > 0.0)) set_error(st, kDevSolveDiag, diag);
      const double inv = 1.0 / diag;
      a.coef[k] = z0 * inv;
      a.coef[a.k + k] = z1 * inv;
      a.coef[2 * a.k + k] = z2 * inv;
      const double f = a.lam_num[k] * inv;
      a.g4[k] = make_float4(static_cast<float>(z0 * f), static_cast<float>(z1 * f),
                            static_cast<float>(z2 * f), 0.f);
    }
    if (c == 0 && tid == 0) st->sigma2_m = sigma2;
  }
  grid.sync();
  SMALL_PROBE(7);

  // ---- phase 3: V = Q g on the row slice, transform, σ² terms.  Threads =
  // (row group, slot) as in phase 1; the CTA walks its rows in chunks of
  // 8·ng rows: every thread has 8 row loads in flight, writes its fp32
  // partial dot products to shared memory, then one thread per row sums the
  // slots in order (fp64) and finalises the row (transform_sigma_kernel).
  // [component][slot][row in chunk], rows padded to an odd stride: the
  // per-row reduction reads consecutive words across threads
  float* vp = reinterpret_cast<float*>(fused_smem);
  if (a.stamps && c == 0 && tid == 0) a.stamps[4 * it + 2] = globaltimer();
  // g in shared memory as [i][quad] (i = column within the quad): one L2 read
  // per CTA, conflict-free reads across consecutive quads
  float4* g4s = reinterpret_cast<float4*>(fused_smem + kFusedSmem);
  const bool use_g4s = keff <= kG4Max;
  if (use_g4s) {
    for (int k = tid; k < keff; k += kFusedThreads) g4s[(k & 3) * nq + (k >> 2)] = __ldcg(a.g4 + k);
    __syncthreads();
  }
  __shared__ double wsum[kFusedWarps];
  {
    const int S = nq < kFusedThreads ? nq : kFusedThreads;  // slots
    const int ng = kFusedThreads / S;
    const int grp = tid / S, slot = tid % S;
    const bool on = grp < ng;
    const int rc = 8 * ng;  // rows per chunk
    // lanes per row in the slot reduction: all the threads over the chunk's
    // rows (a power of two ≤ 32: C1 4 lanes × 12 slots, C0 32 × 16)
    int red_lanes = 1;
    while (red_lanes < 32 && 2 * red_lanes * rc <= kFusedThreads) red_lanes *= 2;
    const int rcp = rc | 1;  // padded row stride of the partials
    const int64_t ld4 = a.kpad / 4;
    const float4* qrow = reinterpret_cast<const float4*>(a.q);
    double term_t = 0.0;  // this thread's σ² terms (rows it finalises), in row order
    for (int64_t cb = r0; cb < r1; cb += rc) {
      if (on) {
        float3 f[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) f[w] = make_float3(0.f, 0.f, 0.f);
        for (int q = slot; q < nq; q += S) {
          float4 qv[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const int64_t r = cb + grp + int64_t(w) * ng;
            qv[w] = r < r1 ? __ldg(qrow + r * ld4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          float4 gk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)  // written in phase 2
            gk[i] = use_g4s ? g4s[i * nq + q] : __ldcg(a.g4 + 4 * q + i);
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const float qq[4] = {qv[w].x, qv[w].y, qv[w].z, qv[w].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              f[w].x = __fmaf_rn(qq[i], gk[i].x, f[w].x);
              f[w].y = __fmaf_rn(qq[i], gk[i].y, f[w].y);
              f[w].z = __fmaf_rn(qq[i], gk[i].z, f[w].z);
            }
          }
        }
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          float* v = vp + slot * rcp + grp + w * ng;
          v[0] = f[w].x;
          v[S * rcp] = f[w].y;
          v[2 * S * rcp] = f[w].z;
        }
      }
      __syncthreads();
      // L threads per row sum interleaved slots (fp64), combined by a fixed
      // xor tree; the group's first lane finalises the row
      const int L = red_lanes, rows_per_pass = kFusedThreads / L;
      for (int pass = 0; pass * rows_per_pass < rc; ++pass) {  // uniform trip count
        const int rr = pass * rows_per_pass + tid / L;
        const int64_t i = cb + rr;
        const bool live = rr < rc && i < r1;
        const int sub = tid % L;
        double o0 = 0.0, o1 = 0.0, o2 = 0.0, x00 = 0.0, x01 = 0.0, x02 = 0.0;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, vr = 0.0;
        if (live && sub == 0) {  // row data, in flight during the reduction
          o0 = a.xt64[i], o1 = a.xt64[m + i], o2 = a.xt64[2 * m + i];
          x00 = a.x0[i], x01 = a.x0[m + i], x02 = a.x0[2 * m + i];
          p0 = a.ptilde_y[i], p1 = a.ptilde_y[m + i], p2 = a.ptilde_y[2 * m + i];
          vr = a.var[i];
        }
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        if (live)
          for (int j = sub; j < S; j += L) {
            const float* v = vp + j * rcp + rr;
            v0 += v[0];
            v1 += v[S * rcp];
            v2 += v[2 * S * rcp];
          }
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
          v0 += __shfl_xor_sync(0xffffffffu, v0, o);
          v1 += __shfl_xor_sync(0xffffffffu, v1, o);
          v2 += __shfl_xor_sync(0xffffffffu, v2, o);
        }
        if (!live || sub != 0) continue;
        const double n0 = x00 + v0, n1 = x01 + v1, n2 = x02 + v2;
        const double e0 = n0 - o0, e1 = n1 - o1, e2 = n2 - o2;
        const double b0 = p0 - o0, b1 = p1 - o1, b2 = p2 - o2;
        term_t += vr - 2.0 * (e0 * b0 + e1 * b1 + e2 * b2) + (e0 * e0 + e1 * e1 + e2 * e2);
        if (a.xt_prev) {
          a.xt_prev[i] = o0;
          a.xt_prev[m + i] = o1;
          a.xt_prev[2 * m + i] = o2;
        }
        a.xt64[i] = n0;
        a.xt64[m + i] = n1;
        a.xt64[2 * m + i] = n2;
        a.xt4[i] = make_float4(static_cast<float>(n0), static_cast<float>(n1),
                               static_cast<float>(n2), 0.f);
      }
      __syncthreads();  // vp is rewritten by the next chunk
    }
    SMALL_PROBE(8);
    const double tw = warp_sum(term_t);  // fixed xor tree
    if (lane == 0) wsum[warp] = tw;
    __syncthreads();
    __shared__ int is_last;
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < kFusedWarps; ++w) sum += wsum[w];
      a.sig_part[c] = sum;
      __threadfence();
      is_last = atomicAdd(a.done, 1) == G - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
  }

  // ---- phase 4 (the last CTA to finish phase 3): σ² (sigma_final_kernel)
  if (tid == 0) *a.done = 0;  // self-resetting for the next replay
  double s = 0.0;
  for (int b = tid; b < G; b += kFusedThreads) s += __ldcg(a.sig_part + b);
  s = warp_sum(s);
  __shared__ double fin[kFusedWarps];
  if (lane == 0) fin[warp] = s;
  __syncthreads();
  if (tid != 0) return;
  double tot = 0.0;
  for (int w = 0; w < kFusedWarps; ++w) tot += fin[w];
#ifdef FCPD_SMALL_PROBE
  if (st->iter == 5) {
    const unsigned long long t9 = globaltimer();
    printf("[probe] pass1 %.2f sync %.2f pass2 %.2f mphase1 %.2f sync %.2f phase2+sync %.2f phase3 %.2f tail %.2f us\n",
           1e-3 * (g_probe[1] - g_probe[0]), 1e-3 * (g_probe[2] - g_probe[1]),
           1e-3 * (g_probe[3] - g_probe[2]), 1e-3 * (g_probe[5] - g_probe[4]),
           1e-3 * (g_probe[6] - g_probe[5]), 1e-3 * (g_probe[7] - g_probe[6]),
           1e-3 * (g_probe[8] - g_probe[7]), 1e-3 * (t9 - g_probe[8]));
  }
#endif
  finish_iteration_sigma(st, tot, m, a.d, a.early_stop, a.trace, a.stamps);
}

__global__ void __launch_bounds__(kFusedThreads, 1) mstep_fused_kernel(MstepFusedArgs a) {
  griddep_wait();
  mstep_fused_body(a);
}

// ===========================================================================
// Small problems (C0: M = N = 2000): the whole EM iteration as ONE
// cooperative kernel.  On the stream-K pass kernels such a problem is all
// latency: 4 M pairs per pass are ~1 µs of MUFU time, but five launches
// (pass 1, its combine, pass 2, its combine, the fused M-step) with their
// global round trips took ~50 µs per iteration.  Here each CTA owns whole
// columns in pass 1 and whole rows in pass 2, so neither pass needs a
// cross-CTA combine:
//   pass 1  CTA c: scene columns [c·N/G, (c+1)·N/G); the model (scaled) in
//           shared memory; a warp per column, lanes over m: fp32 runs of
//           ≤ 64 terms → fp64, fixed xor tree; b_n = −log2(Σ + c) as
//           col_finalize, or the exact max-shifted sum (col_fallback) when
//           the mass is below the flush-to-zero guard
//   — grid sync —
//   pass 2  CTA c: model rows [c·M/G, (c+1)·M/G) — the fused M-step's row
//           slice; the scene (scaled, b in .w) in shared memory; a warp per
//           row: S0, Σw·y', Σw·t (difference form), finalize_row, or the
//           exact row fallback; R = P̃Y − X for the CTA's own rows
//   M-step  mstep_fused_body: its z partials read only the CTA's own rows
//           of R (no grid sync before it), then its own two syncs.
// Three grid syncs and one launch per iteration.  Pairs are evaluated in the
// difference form (the pass kernels' exact path; the centred form is a
// throughput device that does not matter here).
namespace {
constexpr int kSmallRun = 64;  // fp32 run length of the per-lane sums before fp64
constexpr int kSmallMaxPts = 8192;  // the staged set (128 KB, as packed pairs)
constexpr int kSmallPtsBytes = kSmallMaxPts * 16;
static_assert(kSmallPtsBytes <= kFusedDynSmem, "small iteration fits the fused M-step's smem");
// padding point of an odd count: t ≈ 3e37 (2^-t = 0), b = −∞ (weight 0)
#define kSmallPad make_float4(3.0e18f, 3.0e18f, 3.0e18f, -INFINITY)
// point i of the packed-pair staging
__device__ __forceinline__ float4 small_pt(const float4* pa, const float4* pb, int64_t i) {
  const float4 A = pa[i >> 1], B = pb[i >> 1];
  return (i & 1) ? make_float4(A.y, A.w, B.y, B.w) : make_float4(A.x, A.z, B.x, B.z);
}

}  // namespace

__global__ void __launch_bounds__(kFusedThreads, 1) small_iter_kernel(SmallIterArgs a) {
  const MstepFusedArgs& ms = a.ms;
  IterState* st = ms.st;
  if (!st->active) return;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t m = ms.m, n = a.n;
  if (ms.stamps && c == 0 && tid == 0) ms.stamps[4 * st->iter] = globaltimer();
  extern __shared__ __align__(16) unsigned char fused_smem[];
  const float s = st->sx;

  SMALL_PROBE(0);
  // ---- pass 1: b_n of the CTA's scene columns.  A warp per column, lanes
  // over packed pairs of model points (f32x2: 7 FP32 ops and 2 ex2 per two
  // pairs), two pairs of pairs in flight per lane; fp32 runs of ≤ 64 terms
  // per lane element, then fp64 and a fixed xor tree.
  float4* pa = reinterpret_cast<float4*>(fused_smem);                   // (x0,x1,y0,y1)
  float4* pb = reinterpret_cast<float4*>(fused_smem + kSmallPtsBytes / 2);  // (z0,z1,b0,b1)
  const int64_t mp = (m + 1) / 2;
  for (int64_t k = tid; k < mp; k += kFusedThreads) {
    const float4 p0 = scale_pt(ms.xt4[2 * k], s);
    const float4 p1 = 2 * k + 1 < m ? scale_pt(ms.xt4[2 * k + 1], s) : kSmallPad;
    pa[k] = make_float4(p0.x, p1.x, p0.y, p1.y);
    pb[k] = make_float4(p0.z, p1.z, 0.f, 0.f);
  }
  __syncthreads();
  {
    const double log2c = st->log2c;
    const double cst = exp2(log2c);  // 0 when ω = 0
    const int64_t n0 = c * n / G, n1 = (c + 1) * n / G;
    for (int64_t col = n0 + warp; col < n1; col += kFusedWarps) {
      const float4 yv = scale_pt(a.y4b[col], s);
      const float2 nx = make_float2(-yv.x, -yv.x), ny = make_float2(-yv.y, -yv.y),
                   nz = make_float2(-yv.z, -yv.z), m1 = make_float2(-1.f, -1.f);
      double tot = 0.0;
      float2 f0 = make_float2(0.f, 0.f), f1 = f0;
      int run = 0;
      auto pair = [&](int64_t k, float2& f) {
        const float4 A = pa[k], B = pb[k];
        const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx);
        const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny);
        const float2 dz = __fadd2_rn(make_float2(B.x, B.y), nz);
        float2 t = __fmul2_rn(dx, dx);
        t = __ffma2_rn(dy, dy, t);
        t = __ffma2_rn(dz, dz, t);
        t = __fmul2_rn(t, m1);
        f = __fadd2_rn(f, make_float2(ex2_approx(t.x), ex2_approx(t.y)));
      };
      int64_t k = lane;
      for (; k + 32 < mp; k += 64) {
        pair(k, f0);
        pair(k + 32, f1);
        if (++run == kSmallRun / 2) {
          tot += static_cast<double>(f0.x) + f0.y + f1.x + f1.y;
          f0 = f1 = make_float2(0.f, 0.f);
          run = 0;
        }
      }
      if (k < mp) pair(k, f0);
      tot = warp_sum(tot + static_cast<double>(f0.x) + f0.y + f1.x + f1.y);
      double b2;
      if (tot + cst >= static_cast<double>(m) * 0x1p-76) {  // col_finalize
        b2 = -log2(tot + cst);
      } else {  // exact: max-shifted fp64 (col_fallback)
        float tmin = INFINITY;
        for (int64_t i = lane; i < m; i += 32) tmin = fminf(tmin, sqdist(yv, small_pt(pa, pb, i)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
        double shift = -static_cast<double>(tmin);
        if (log2c > shift) shift = log2c;
        double e = 0.0;
        for (int64_t i = lane; i < m; i += 32)
          e += exp2(-static_cast<double>(sqdist(yv, small_pt(pa, pb, i))) - shift);
        e = warp_sum(e);
        const double cc = log2c > -INFINITY ? exp2(log2c - shift) : 0.0;
        b2 = -(shift + log2(e + cc));
      }
      if (lane == 0) {
        a.b2[col] = b2;
        a.y4b[col].w = static_cast<float>(b2);
      }
    }
  }
  SMALL_PROBE(1);
  grid.sync();
  SMALL_PROBE(2);

  // ---- pass 2: the CTA's model rows (the M-step's row slice).  A warp per
  // row, lanes over packed pairs of scene points: L = b − t, w = 2^L, sums
  // S0, Σw·y' (3), Σw·t (12 FP32 ops and 2 ex2 per two pairs)
  const int64_t np2 = (n + 1) / 2;
  for (int64_t k = tid; k < np2; k += kFusedThreads) {
    const float4 p0 = scale_pt(__ldcg(a.y4b + 2 * k), s);
    const float4 p1 = 2 * k + 1 < n ? scale_pt(__ldcg(a.y4b + 2 * k + 1), s) : kSmallPad;
    pa[k] = make_float4(p0.x, p1.x, p0.y, p1.y);
    pb[k] = make_float4(p0.z, p1.z, p0.w, p1.w);
  }
  __syncthreads();
  {
    const double sc = derived_scale(st);
    const int64_t r0 = c * m / G, r1 = (c + 1) * m / G;
    for (int64_t row = r0 + warp; row < r1; row += kFusedWarps) {
      const float4 xv = scale_pt(ms.xt4[row], s);
      const float2 nx = make_float2(-xv.x, -xv.x), ny = make_float2(-xv.y, -xv.y),
                   nz = make_float2(-xv.z, -xv.z);
      double d[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      float2 f[2][5];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 5; ++q) f[h][q] = make_float2(0.f, 0.f);
      auto pair = [&](int64_t k, float2 (&g)[5]) {
        const float4 A = pb[k], X = pa[k];
        const float2 yx = make_float2(X.x, X.y), yy = make_float2(X.z, X.w);
        const float2 yz = make_float2(A.x, A.y), bb = make_float2(A.z, A.w);
        const float2 dx = __fadd2_rn(yx, nx), dy = __fadd2_rn(yy, ny), dz = __fadd2_rn(yz, nz);
        float2 t = __fmul2_rn(dx, dx);
        t = __ffma2_rn(dy, dy, t);
        t = __ffma2_rn(dz, dz, t);
        const float2 L = __ffma2_rn(t, make_float2(-1.f, -1.f), bb);
        const float2 w = make_float2(ex2_approx(L.x), ex2_approx(L.y));
        g[0] = __fadd2_rn(g[0], w);
        g[1] = __ffma2_rn(w, yx, g[1]);
        g[2] = __ffma2_rn(w, yy, g[2]);
        g[3] = __ffma2_rn(w, yz, g[3]);
        g[4] = __ffma2_rn(w, t, g[4]);
      };
      auto drain = [&]() {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          d[q] += static_cast<double>(f[0][q].x) + f[0][q].y + f[1][q].x + f[1][q].y;
          f[0][q] = f[1][q] = make_float2(0.f, 0.f);
        }
      };
      int run = 0;
      int64_t k = lane;
      for (; k + 32 < np2; k += 64) {
        pair(k, f[0]);
        pair(k + 32, f[1]);
        if (++run == kSmallRun / 2) {
          drain();
          run = 0;
        }
      }
      if (k < np2) pair(k, f[0]);
      drain();
#pragma unroll
      for (int q = 0; q < 5; ++q) d[q] = warp_sum(d[q]);
      double log2p1;
      if (d[0] >= static_cast<double>(n) * 0x1p-76) {
        log2p1 = log2(d[0]);
      } else {  // exact: max-shifted fp64 (row_fallback)
        float lmax = -INFINITY;
        for (int64_t j = lane; j < n; j += 32) {
          const float4 yv = small_pt(pa, pb, j);
          lmax = fmaxf(lmax, yv.w - sqdist(yv, xv));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
#pragma unroll
        for (int q = 0; q < 5; ++q) d[q] = 0.0;
        if (lmax > -INFINITY) {
          for (int64_t j = lane; j < n; j += 32) {
            const float4 yv = small_pt(pa, pb, j);
            const float t = sqdist(yv, xv);
            const double wgt = exp2(static_cast<double>(yv.w - t) - static_cast<double>(lmax));
            d[0] += wgt;
            d[1] += wgt * yv.x;
            d[2] += wgt * yv.y;
            d[3] += wgt * yv.z;
            d[4] += wgt * t;
          }
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) d[q] = warp_sum(d[q]);
        log2p1 = d[0] > 0 ? static_cast<double>(lmax) + log2(d[0]) : -INFINITY;
      }
      if (lane == 0)
        finalize_row(row, m, log2p1, d[0], d[1], d[2], d[3], d[4], ms.xt64, sc, a.out, a.ys, st);
    }
  }
  if (c == 0 && tid == 0 && a.counters) {  // every pair evaluated, difference form
    // (tile pairs are counted by culling sessions only, as on the pass kernels)
    const unsigned long long pairs = static_cast<unsigned long long>(m) * n;
    atomicAdd(a.counters + 3, pairs);
    atomicAdd(a.counters + 5, pairs);
  }
  SMALL_PROBE(3);
  __syncthreads();  // the CTA's rows of R (and P̃Y, var) are written; the
                    // M-step's z partials read exactly these rows
  mstep_fused_body(ms);
}

bool small_iter_fits(int64_t m, int64_t n) {
  return m <= kSmallMaxPts && n <= kSmallMaxPts && m * n <= (int64_t(1) << 24);
}

void launch_small_iter(const SmallIterArgs& args, int grid, cudaStream_t stream) {
  FCPD_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(&small_iter_kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedDynSmem));
  SmallIterArgs a = args;
  void* params[] = {&a};
  FCPD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&small_iter_kernel),
                                        dim3(grid), dim3(kFusedThreads), params, kFusedDynSmem,
                                        stream));
}

int mstep_fused_grid(int sm_count) { return sm_count; }

void launch_mstep_fused(const MstepFusedArgs& args, int grid, cudaStream_t stream) {
  // per launch: the attribute belongs to the current device
  FCPD_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(&mstep_fused_kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedDynSmem));
  MstepFusedArgs a = args;
  void* params[] = {&a};
  FCPD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&mstep_fused_kernel),
                                        dim3(grid), dim3(kFusedThreads), params, kFusedDynSmem,
                                        stream));
}

}  // namespace fcpd
