// estep.cuh — E-step launch interface (see estep.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace fcpd {

// one column pair / row pair per thread: a 128-thread CTA covers exactly one
// 256-point tile, the culling granularity
constexpr int kColsPerThread = 2;
constexpr int kRowsPerThread = 2;
constexpr int kMaxRowChunks = 8;  // pass-2 row chunks (overlap with the Qᵀ·R stream)

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

struct EStepPlan {
  int col_blocks = 0, col_splits = 0;
  int64_t m_per_split = 0;
  int row_blocks = 0, row_splits = 0;
  int64_t n_per_split = 0;
  // per-chunk pass-2 splits when pass 2 runs as row chunks (overlap form):
  // fewer row blocks per launch need more N-splits to fill the GPU
  int chunks = 1;
  int chunk_splits[kMaxRowChunks] = {};
  int64_t chunk_nps[kMaxRowChunks] = {};
  int max_row_splits() const {
    int s = row_splits;
    for (int c = 0; c < chunks; ++c) s = chunk_splits[c] > s ? chunk_splits[c] : s;
    return s;
  }
};
void plan_row_chunks(EStepPlan& p, int64_t m, int64_t n, int sm_count, int chunks);

// Tile culling.  Points are Morton-sorted by the engine
// so 256-point tiles are compact boxes; a (column block, model tile) or (row
// block, scene tile) pair is skipped when every pair term in it is below
// 2^-margin of the smallest possible column (row) total.  With margin =
// 50 + log2(count) the skipped mass is ≤ 2^-50 relative: exact to fp32.
struct CullInfo {
  int enabled = 0;
  int n_xtiles = 0, n_ytiles = 0;   // 256-point tiles
  const float4* xlo = nullptr;      // model tiles (x̃ of this iteration)
  const float4* xhi = nullptr;
  const float4* ylo = nullptr;      // scene tiles (fixed)
  const float4* yhi = nullptr;
  const float* col_bound = nullptr; // per scene tile: U (unscaled d²)
  const float* row_bound = nullptr; // per model tile: lower bound of max L (log2)
  const float2* bminmax = nullptr;  // per scene tile: (min b, max b)
  float margin1 = 0.f, margin2 = 0.f;
  unsigned long long* counters = nullptr;  // [0] pass-1 tiles, [1] pass-2 tiles evaluated
};

struct CullBuffers {  // writable views of the CullInfo arrays (engine-owned)
  float4 *xlo, *xhi, *ylo, *yhi;
  float *col_bound, *row_bound;
  float2* bminmax;
};

struct EStepBuffers {
  const float4* xt4;   // x̃ fp32 (x,y,z,0), M
  const double* xt64;  // x̃ fp64 SoA M×3
  float4* y4b;         // y fp32 (x,y,z,b2), N — .w written by pass 1
  double* b2;          // b_n fp64 (log2 units), N
  double* pt1;         // optional Σ_m P_mn, N
  double* col_part;    // [col_splits][N]
  double* row_part;    // [row_splits][5][M]
  int32_t* col_flags;  // N
  int32_t* row_flags;  // M
  int32_t* flags_count;  // 2
  RowOut out;
  YStats ystats;
  CullInfo cull;      // cull.enabled = 0 → dense (every pair evaluated)
  CullBuffers cullw;  // geometry buffers written each iteration
};

// Scene-tile boxes (once per session; Y does not move).
void launch_tile_bbox(const float4* pts, int64_t count, float4* lo, float4* hi,
                      const IterState* st, cudaStream_t stream);

EStepPlan make_estep_plan(int64_t m, int64_t n, int sm_count);
// Pieces of launch_estep for the distributed path (n = local scene count;
// the prologue's outlier constant uses the global N).
void launch_estep_prologue(IterState* st, int64_t m, int64_t n_global, int d, double omega,
                           int32_t* flags_count, uint64_t* stamps, cudaStream_t stream);
void launch_estep_pass1(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                        IterState* st, cudaStream_t stream);
void launch_estep_pass2_partials(const EStepPlan& p, const EStepBuffers& b, int64_t m,
                                 int64_t n, IterState* st, cudaStream_t stream);

struct RowChunk {
  int rb0 = 0, rb1 = 0;      // row blocks
  int64_t r0 = 0, r1 = 0;    // model rows
};
RowChunk row_chunk(const EStepPlan& p, int64_t m, int c, int chunks);
void launch_estep_pass2_chunk(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n,
                              IterState* st, cudaStream_t stream, int c, int chunks);
void launch_estep(const EStepPlan& p, const EStepBuffers& b, int64_t m, int64_t n, int d,
                  double omega, IterState* st, uint64_t* stamps, cudaStream_t stream,
                  cudaEvent_t mid = nullptr);

}  // namespace fcpd
