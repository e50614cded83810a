// common.cuh — shared device helpers for the B200 Fast-CPD hot path.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "fcpd_capi.h"

namespace fcpd {

// Error carried from the engine to the C-ABI boundary; `code` is one of the
// FCPD_ERR_* values of include/fcpd_capi.h.
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FCPD_CUDA(call)                                                         \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      throw ::fcpd::Failure(e_ == cudaErrorMemoryAllocation ? FCPD_ERR_OOM       \
                                                            : FCPD_ERR_CUDA,     \
                            std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define FCPD_LAUNCH_CHECK() FCPD_CUDA(cudaGetLastError())

constexpr double kSigma2Floor = 1e-10;      // correspondence.hpp:12
constexpr double kLog2e = 1.4426950408889634;
// log2(1e-300): rows whose raw posterior mass is below 1e-300 fall back to
// the uniform row (correspondence.hpp:89).
constexpr double kLog2DegenerateRow = -996.5784284662087;

// Device error slots (first error wins).  Codes mirror the reference's
// NumericError sites so the host can rebuild the reference message.
enum DevErr : int {
  kDevOk = 0,
  kDevSolveDiag = 1,    // solvers.hpp:68-69
  kDevNegVariance = 2,  // solvers.hpp:173-174
};

// Per-iteration scalars living in device memory so a captured CUDA graph can
// replay iterations without host round trips.  The E-step scalars of
// iteration i+1 (σ² floor, coordinate scale, outlier constant) are set by the
// last step of iteration i (estep_scalars_for_next), those of iteration 0 by
// init_state_kernel — there is no per-iteration prologue launch.
struct IterState {
  double sigma2;        // σ² entering this iteration (unclamped, as the reference)
  double sigma2_e;      // max(σ², 1e-10): the value the E-step uses
  double log2c;         // outlier constant in log2 units (only if ω>0)
  float sx;             // sqrt(log2e / (2 σ²_e)): coordinate pre-scale
  float pad0;
  int32_t active;       // 0 after early stop → kernels return immediately
  int32_t iter;         // iteration index
  int32_t err_code;
  int32_t err_iter;
  double err_value;
  int64_t degenerate_rows;  // cumulative
  int64_t sigma2_clamps;    // cumulative
  int32_t iters_run;
  int32_t keff;         // leading eigenpairs the M-step streams this iteration (mstep.cu)
  double sigma2_m;      // σ² the last M-step solved with (final coefficients)
  double sigma2_e_last; // σ²_e of the last E-step that ran (dense correspondence output)
  // E-step constants (set once by the host): ω, M, global N, D
  double omega;
  int64_t m_all, n_all;
  int32_t dim;
  int32_t flag_count[2];  // columns / rows queued for the exact fallback this iteration
  int32_t cull_on;        // this iteration builds culled work lists (else: every pair)
  int32_t cull_pays;      // the last lists dropped enough units to pay for themselves
  int32_t cull_recheck;   // iterations between list re-checks while they do not pay
};

// Culling lists are built in an iteration when the previous lists dropped
// any unit (kept < kCullKeepFrac of them: σ² only falls, so a culling that
// starts to bite soon pays for its list kernels), else only every
// IterState::cull_recheck-th iteration: 1 where the list kernels are a small
// share of a pass (C3/C4: tens of ms of pairs), kCullRecheck otherwise (C1's
// first iterations: nothing to drop, lists ≈ 3 % of an iteration).
constexpr int kCullRecheck = 4;
constexpr double kCullKeepFrac = 0.999;

// The E-step scalars for σ² (correspondence.hpp:43-47 floor + clamp flag,
// :61-66 outlier constant in log2 units), the fallback queues emptied, and
// the culling decision — run by ONE thread at the end of an iteration (for
// the next one) and by init_state_kernel (iteration 0).
__device__ __forceinline__ void estep_scalars_for_next(IterState* st, double sigma2, int next_iter) {
  st->sigma2_e_last = st->sigma2_e;
  double s2 = sigma2;
  if (s2 < kSigma2Floor) {
    s2 = kSigma2Floor;
    st->sigma2_clamps += 1;
  }
  st->sigma2_e = s2;
  st->sx = static_cast<float>(sqrt(kLog2e / (2.0 * s2)));
  if (st->omega > 0.0) {
    const double log_c = 0.5 * st->dim * log(2.0 * M_PI * s2) +
                         log(st->omega / (1.0 - st->omega)) +
                         log(static_cast<double>(st->m_all) / static_cast<double>(st->n_all));
    st->log2c = log_c * kLog2e;
  } else {
    st->log2c = -INFINITY;
  }
  st->flag_count[0] = st->flag_count[1] = 0;
  st->cull_on = next_iter == 0 || st->cull_pays ||
                next_iter % (st->cull_recheck > 0 ? st->cull_recheck : kCullRecheck) == 0;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (PDL).  Hot-path kernels are launched with
// launch_pdl: the next kernel in the stream (graph) may be scheduled while
// its predecessor drains, hiding the launch gap.  Such a kernel must call
// griddep_wait() before touching anything its predecessor writes — every
// kernel launched this way does so as its first statement (a no-op when it
// was launched normally).
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // let the next kernel be scheduled now: its CTAs become resident as ours
  // retire and block in their own wait until this grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();  // FCPD_PDL=0 → ordinary launches (engine.cu)

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FCPD_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

__device__ __forceinline__ void set_error(IterState* st, int code, double value) {
  if (atomicCAS(&st->err_code, 0, code) == 0) {
    st->err_iter = st->iter;
    st->err_value = value;
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

}  // namespace fcpd
