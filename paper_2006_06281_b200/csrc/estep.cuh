// estep.cuh — E-step launch interface (see estep.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace fcpd {

constexpr int kTilePts = 256;  // points per tile (a CTA's own block, a staging chunk)
// points per sub-tile: the culling unit of the other set (the engine's k-d
// order makes every 32-point sub-tile of a 256-point tile a compact box)
constexpr int kSubPts = 32;
constexpr int kSubPerTile = kTilePts / kSubPts;

// Fallback-path per-row outputs (all device pointers; SoA fp64 M×3).
struct RowOut {
  double* ptilde_y;   // (P̃Y)_m
  double* var;        // Σ_n P̃_mn ‖y_n − x̃_m‖²
  double* log2p1;     // log2 of the raw row mass Σ_n P_mn
  int32_t* degenerate;
  float4* resid4;     // optional: R = P̃Y − X for the M-step (fp32)
  const double* x0;   // X (normalised model) when resid4 is set
};

// Statistics of the scene for the uniform-row fallback (fp64).
struct YStats {
  double mean[3];
  double sq_mean;
};

// The work of one pass: for each of n_blocks own 256-point blocks (scene
// tiles in pass 1, model tiles in pass 2), the list of units of the other
// set whose pairs are evaluated.  A unit is upts() consecutive points of the
// other set (a 32-point sub-tile; 256-point tiles for the tensor-core pass
// 2).  Entries = (block, unit) pairs in block-major order; offset[b] =
// entries before block b.  implicit = every unit of every block (no
// culling): tiles/offset are not read.
struct WorkList {
  int implicit = 1;
  int n_blocks = 0, n_other = 0;  // n_other = units of the other set
  int ushift = 5;                 // points per unit = 1 << ushift (kSubPts)
  const int32_t* tiles = nullptr;   // [n_blocks][n_other]
  const int32_t* offset = nullptr;  // [n_blocks + 1]
  // culling sessions: the list is used only when *dyn_on (IterState::cull_on,
  // decided per iteration); otherwise the pass is implicit and adds its
  // n_blocks·n_other units to *implicit_counter (tiles_evaluated)
  const int32_t* dyn_on = nullptr;
  unsigned long long* implicit_counter = nullptr;
  __host__ __device__ int64_t off(int b) const {
    return implicit ? static_cast<int64_t>(b) * n_other : static_cast<int64_t>(offset[b]);
  }
  __host__ __device__ int upts() const { return 1 << ushift; }
  __host__ __device__ int tile(int b, int64_t k) const {
    return implicit ? static_cast<int>(k) : tiles[static_cast<int64_t>(b) * n_other + k];
  }
};

struct WorkListBuffers {  // writable views (engine-owned)
  int32_t* tiles = nullptr;
  int32_t* offset = nullptr;
  int32_t* done = nullptr;     // last-CTA counter of the list kernel (self-resetting)
};

// Persistent stream-K schedule of both passes (one CTA wave per pass).
// Blocks whose squared box half-diagonal in the scaled frame exceeds this run
// in the difference form (the centred form's rounding ≈ 4ε·R² in log2
// units; 16 → ≤ 4e-6).
constexpr float kCentredMaxR2 = 16.f;

struct EStepPlan {
  int centred = 1;  // tile-centred pair form where exact enough; FCPD_ESTEP_FORM=diff → off
  float centred_max_r2 = kCentredMaxR2;  // per-segment guard (< 0: difference form only)
  int row_pairs = 2;  // pass 2: packed row pairs per thread (FCPD_ROW_PAIRS=1 → 1)
  int col_pairs = 2;  // pass 1: packed column pairs per thread (FCPD_COL_PAIRS=1 → 1)
  int flush2 = 64;  // fp32 run length of the pass-2 sums (FCPD_FLUSH2, power of two)
  int ex2_poly = 1;  // pass 1: of every 8 staged points, this many take ex2 on the FMA pipe (FCPD_EX2_POLY)
  int col_minb = 16;  // pass 1: CTAs per SM, 16 or 32 (large passes; FCPD_COL_MINB)
  int col_blocks = 0, row_blocks = 0;  // scene tiles (pass-1 blocks), model tiles (pass 2)
  int col_grid = 0, row_grid = 0;      // persistent CTAs per pass
  size_t col_seg_doubles() const { return static_cast<size_t>(col_grid + col_blocks) * kTilePts; }
  size_t row_seg_doubles() const {
    return static_cast<size_t>(row_grid + row_blocks) * 5 * kTilePts;
  }
};

// Tile culling.  Points are k-d sorted by the engine so
// 256-point tiles and their 32-point sub-tiles are compact boxes; a (block,
// sub-tile) pair is dropped from the work list when every pair term in it
// is below 2^-margin of the
// smallest possible column (row) total.  With margin = bits + log2(count)
// the skipped mass is ≤ 2^-bits relative (engine.cu: 32 bits).  The lower
// bound on the totals comes from box geometry and, with `probe`, from exact
// nearest-point distances to the two closest tiles (estep.cu list kernels).
struct CullInfo {
  int enabled = 0;  // culling drops tile pairs from the work lists
  int probe = 1;    // probe bound on (FCPD_CULL_PROBE=0 → box bound only)
  int lists = 0;    // explicit work lists (culling, or pass-2 routing to tensor cores)
  int n_xtiles = 0, n_ytiles = 0;   // 256-point tiles (own blocks; probe choice)
  int n_xsub = 0, n_ysub = 0;       // 32-point sub-tiles (the culling units)
  const float4* xlo = nullptr;      // model tiles (x̃ of this iteration)
  const float4* xhi = nullptr;
  const float4* ylo = nullptr;      // scene tiles (fixed)
  const float4* yhi = nullptr;
  const float2* bminmax = nullptr;  // per scene tile: (min b, max b)
  const float4* sxlo = nullptr;     // model sub-tiles
  const float4* sxhi = nullptr;
  const float4* sylo = nullptr;     // scene sub-tiles
  const float4* syhi = nullptr;
  const float2* sbminmax = nullptr;  // per scene sub-tile: (min b, max b)
  float margin1 = 0.f, margin2 = 0.f;
  // [0] pass-1, [1] pass-2 work-list entries evaluated, in (256-point block,
  // 32-point sub-tile) pairs; [2..5] pairs evaluated by (pass 1 centred,
  // pass 1 difference, pass 2 centred, pass 2 difference) form — the
  // instruction mix the roofline is computed from
  unsigned long long* counters = nullptr;
  // pass-1 list (read by the pass-2 list kernel for the "culling pays" test)
  const int32_t* wl1_offset = nullptr;
  int64_t wl1_units = 0, wl2_units = 0;  // units of the full (implicit) lists
  // per own block: did the last probe drop ≥ 1/4 of the box-kept tiles?
  // (blocks whose probe does not pay reconsider it every 4th iteration)
  int32_t* probe_paid1 = nullptr;  // [n_ytiles]
  int32_t* probe_paid2 = nullptr;  // [n_xtiles]
};

struct CullBuffers {  // writable views of the CullInfo arrays (engine-owned)
  float4 *xlo, *xhi, *ylo, *yhi;
  float2* bminmax;
  float4 *sxlo, *sxhi, *sylo, *syhi;
  float2* sbminmax;
};

struct EStepBuffers {
  const float4* xt4;   // x̃ fp32 (x,y,z,0), M
  const double* xt64;  // x̃ fp64 SoA M×3
  float4* y4b;         // y fp32 (x,y,z,b2), N — .w written by pass 1
  double* b2;          // b_n fp64 (log2 units), N
  double* pt1;         // optional Σ_m P_mn, N
  double* col_seg;     // pass-1 segment partials [col_grid + col_blocks][256]
  double* row_seg;     // pass-2 segment partials [grid + row_blocks][5][256]
  int32_t* col_done;   // [col_blocks] segment arrival counters (self-resetting)
  int32_t* row_done;   // [row_blocks]
  int32_t* col_flags;  // N: columns queued for the exact fallback
  int32_t* row_flags;  // M
  RowOut out;
  YStats ystats;
  double* row_aos;     // distributed: row sums AoS [m_pad][5] instead of `out`
  CullInfo cull;      // cull.enabled = 0 → implicit work lists (every pair evaluated)
  CullBuffers cullw;  // geometry buffers written each iteration
  WorkListBuffers wl1, wl2;  // pass-1 / pass-2 work lists (used when culling)
  uint64_t* stamps;   // device phase timestamps [iteration][4] (optional)
};

// Tile and sub-tile boxes (scene: once per session, Y does not move).
void launch_tile_bbox(const float4* pts, int64_t count, float4* lo, float4* hi, float4* slo,
                      float4* shi, const IterState* st, cudaStream_t stream);

EStepPlan make_estep_plan(int64_t m, int64_t n, int sm_count);
// Iteration-0 state: E-step scalars of sigma2, ω, M, global N, D (device
// math, the same code the iterations use for the next σ²).
void launch_init_state(IterState* st, double sigma2, double omega, int64_t m, int64_t n_global,
                       int d, cudaStream_t stream);
// Pass 1 (column normalisers; each scene block finalised by the CTA that
// completes it) + the column fallback.  n = local scene count.
void launch_estep_pass1(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream);
// Pass 2: single GPU → finalised rows (b.out) + the exact row fallback;
// distributed (b.row_aos) → per-row sums of the local columns, AoS [m_pad][5].
void launch_estep_pass2(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream);
void launch_estep(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                  IterState* st, cudaStream_t stream, cudaEvent_t mid = nullptr);
// kernels one E-step launches (culling session or not; single GPU or not)
int estep_kernels(bool culling, bool dist);

}  // namespace fcpd
