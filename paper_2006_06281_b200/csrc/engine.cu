// engine.cu — host orchestration + C ABI (include/fcpd_capi.h).
//
// register_pointsets (registration.hpp:79-175) as a device-resident loop:
//   validate → normalize_pair (host, fp64, O(M+N)) → upload →
//   spectral setup (cached per context) → init_sigma2 → one CUDA graph per
//   EM iteration, replayed `iterations` times with no host round trip →
//   one read-back (σ² trace, x̃, W, diagnostics, device phase timestamps).

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "comm.cuh"
#include "common.cuh"
#include "ctx.cuh"
#include "dist.cuh"
#include "estep.cuh"
#include "mstep.cuh"
#include "nccl_dyn.cuh"
#include "setup.cuh"

#define FCPD_NCCL(call)                                                               \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess)                                                            \
      throw ::fcpd::Failure(FCPD_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

namespace fcpd {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    FCPD_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Run f(0..tasks-1) on `tasks` host threads (the caller's included).  Used
// for the O(M+N) host passes of a register call, each task a fixed slice
// (coordinate × point set), so every result is the same as the serial one.
template <typename F>
void parallel_for(int tasks, F f) {
  std::vector<std::thread> th;
  th.reserve(tasks > 1 ? tasks - 1 : 0);
  for (int i = 1; i < tasks; ++i) th.emplace_back(f, i);
  if (tasks > 0) f(0);
  for (auto& t : th) t.join();
}

// Basis-cache key of the (normalised, sorted) model: four independent
// 64-bit multiply-xor lanes over 8-byte words (≈ 8× the byte-wise rate),
// byte-wise FNV-1a for the tail, lanes folded at the end.
uint64_t fnv1a(const void* data, size_t bytes, uint64_t h = 1469598103934665603ull) {
  const unsigned char* c = static_cast<const unsigned char*>(data);
  constexpr uint64_t kMul = 0x9E3779B97F4A7C15ull;
  uint64_t lane[4] = {h, h ^ 0x1ull, h ^ 0x2ull, h ^ 0x3ull};
  size_t i = 0;
  for (; i + 32 <= bytes; i += 32)
    for (int l = 0; l < 4; ++l) {
      uint64_t w;
      std::memcpy(&w, c + i + 8 * l, 8);
      lane[l] = (lane[l] ^ w) * kMul;
      lane[l] ^= lane[l] >> 29;
    }
  for (int l = 0; l < 4; ++l) h = (h ^ lane[l]) * 1099511628211ull;
  for (; i < bytes; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
  }
  return h;
}

// ------------------------------------------------------------- small kernels

// Dense materialisation (small problems, tests, RegistrationResult::
// correspondence): the reference algorithm itself in fp64 on the device —
// posterior (correspondence.hpp:35-79), one warp per scene column with the
// per-column max shift incl. log c; then enforce_row_constraint (:83-98),
// one thread per model row.  Independent of the streaming fp32 hot path.
__global__ void dense_posterior_kernel(const double* __restrict__ xt64, int64_t m,
                                       const double* __restrict__ y64, int64_t n, int d,
                                       double omega, const IterState* __restrict__ st,
                                       double* __restrict__ p) {
  const int lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n) return;
  const double sigma2 = st->sigma2_e_last;  // the σ² (floored) of the last E-step
  const double inv = 1.0 / (2.0 * sigma2);
  const bool has_outlier = omega > 0.0;
  const double log_c = has_outlier ? 0.5 * d * log(2.0 * M_PI * sigma2) +
                                         log(omega / (1.0 - omega)) +
                                         log(static_cast<double>(m) / static_cast<double>(n))
                                   : 0.0;
  double* col = p + j * m;
  double shift = -INFINITY;
  for (int64_t i = lane; i < m; i += 32) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
      const double t = y64[c * n + j] - xt64[c * m + i];
      s += t * t;
    }
    col[i] = -s * inv;
    shift = fmax(shift, col[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) shift = fmax(shift, __shfl_xor_sync(0xffffffffu, shift, o));
  if (has_outlier && log_c > shift) shift = log_c;
  double denom = 0.0;
  for (int64_t i = lane; i < m; i += 32) {
    col[i] = exp(col[i] - shift);
    denom += col[i];
  }
  denom = warp_sum(denom);
  if (has_outlier) denom += exp(log_c - shift);
  for (int64_t i = lane; i < m; i += 32) col[i] /= denom;
}

__global__ void dense_row_constraint_kernel(double* __restrict__ p, int64_t m, int64_t n,
                                            int32_t* __restrict__ degenerate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) s += p[j * m + i];
  const bool deg = s < 1e-300;
  degenerate[i] = deg ? 1 : 0;
  for (int64_t j = 0; j < n; ++j) p[j * m + i] = deg ? 1.0 / static_cast<double>(n) : p[j * m + i] / s;
}

void launch_dense_posterior(const double* xt64, int64_t m, const double* y64, int64_t n, int d,
                            double omega, const IterState* st, int row_constrain,
                            int32_t* degenerate, double* p, cudaStream_t str) {
  dense_posterior_kernel<<<ceil_div(n, 8), 256, 0, str>>>(xt64, m, y64, n, d, omega, st, p);
  FCPD_LAUNCH_CHECK();
  if (row_constrain) {
    dense_row_constraint_kernel<<<ceil_div(m, 128), 128, 0, str>>>(p, m, n, degenerate);
    FCPD_LAUNCH_CHECK();
  }
}

// coefficients c (fp64 SoA 3×K) → float4 rows for the Qᵀ-row stream.
__global__ void pack_coef_kernel(const double* __restrict__ coef, int64_t k,
                                 float4* __restrict__ c4) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < k)
    c4[i] = make_float4(static_cast<float>(coef[i]), static_cast<float>(coef[k + i]),
                        static_cast<float>(coef[2 * k + i]), 0.f);
}

}  // namespace

// ------------------------------------------------------------------ Session

struct Session {
  int64_t m = 0, n = 0;
  int d = 0;
  fcpd_config cfg{};
  int capacity = 0;  // trace slots
  int launched = 0;  // iterations enqueued since session_begin
  int64_t h2d = 0, d2h = 0;  // bytes copied by the current call
  bool ready = false;
  // normalisation record (pointset.hpp:31-43)
  double center[3] = {0, 0, 0};
  double scale = 1.0;
  double sigma2_initial = 0.0;
  double t_setup_host = 0.0, t_eig = 0.0, t_gram = 0.0;
  bool basis_reused = false;

  DevBuf<double> x0, xt64, xt_prev, y64;
  DevBuf<float4> xt4, y4b, resid4, g4;
  DevBuf<double> b2, pt1, col_seg, row_seg, ptilde_y, var, log2p1, zpart, vpart, coef,
      sig_part, trace;
  DevBuf<int32_t> col_flags, row_flags, col_done, row_done, degenerate;
  DevBuf<uint64_t> stamps;
  DevBuf<IterState> st;

  YStats ystats{};
  EStepPlan ep;
  ColsumPlan zp, vp;
  // z = Qᵀ·R as row dot products over the contiguous prefix of Qᵀ's rows
  // (streaming M-step; FCPD_ZPASS=colsum → column sums over Q instead)
  RowdotPlan zr;
  bool rowdot = false;
  double tau = 0.0;  // spectral truncation threshold of the basis streams (0: off)
  bool mfused = false;            // whole M-step as one cooperative kernel (mstep_fused.cu)
  bool small = false;             // whole iteration as one cooperative kernel (small_iter_kernel)
  int mfused_grid = 0;
  DevBuf<double> zpart_fused;     // [K][grid][3]
  DevBuf<int32_t> mfused_done;    // its last-CTA counter
  cudaGraphExec_t graph = nullptr;
  // spatial order (sorted → original index) and tile-culling buffers
  std::vector<int64_t> perm_x, perm_y;
  bool cull = true;
  DevBuf<float4> xlo, xhi, ylo, yhi;      // 256-point tile boxes
  DevBuf<float4> sxlo, sxhi, sylo, syhi;  // 32-point sub-tile boxes (the culling units)
  DevBuf<float2> bminmax, sbminmax;       // per scene tile / sub-tile: b range
  // (block, sub-tile) pairs evaluated (pass 1, pass 2), cumulative
  DevBuf<unsigned long long> cull_counters;
  DevBuf<int32_t> probe_paid;                // culling probe outcome per block (both passes)
  // per-iteration work lists of the two passes (culled (block, sub-tile) pairs)
  DevBuf<int32_t> wl1_tiles, wl1_off, wl2_tiles, wl2_off, wl_done;

  // ---- distributed (NCCL) sharding: scene N split over ranks, model rows
  // [m0, m0+mr) owned by this rank (m_pad = world·mr ≥ M).  In this mode
  // x0/xt64/xt_prev/ptilde_y/var/log2p1/degenerate/resid4 hold OWN rows
  // (stride mr); xt4 holds all M_pad rows; y4b the local scene shard.
  bool dist = false;
  int64_t n_global = 0, m_pad = 0, mr = 0, m0 = 0, m_valid_own = 0, mr4 = 0;
  DevBuf<double> rowsum_all, rowsum_own, fsum_all, fsum_own, zfull, zcorr, sig_local, stage;
  bool dist_conditional = false;  // the fallback exchange sits in a conditional graph node
  DevBuf<int32_t> mask_own, mask_all;
  DevBuf<float> fmax_all, qt_own;

  void release_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
  }
  void release() {
    release_graph();
    for (auto* b : {&x0, &xt64, &xt_prev, &y64, &b2, &pt1, &col_seg, &row_seg, &ptilde_y,
                    &var, &log2p1, &zpart, &vpart, &coef, &sig_part, &trace, &zpart_fused})
      b->release();
    for (auto* b : {&xt4, &y4b, &resid4, &g4}) b->release();
    for (auto* b : {&col_flags, &row_flags, &col_done, &row_done, &degenerate, &mfused_done})
      b->release();
    stamps.release();
    st.release();
    for (auto* b : {&rowsum_all, &rowsum_own, &fsum_all, &fsum_own, &zfull, &zcorr, &sig_local,
                    &stage})
      b->release();
    mask_own.release();
    mask_all.release();
    fmax_all.release();
    qt_own.release();
    for (auto* b : {&xlo, &xhi, &ylo, &yhi, &sxlo, &sxhi, &sylo, &syhi}) b->release();
    bminmax.release();
    sbminmax.release();
    cull_counters.release();
    probe_paid.release();
    for (auto* b : {&wl1_tiles, &wl1_off, &wl2_tiles, &wl2_off, &wl_done}) b->release();
  }
};

}  // namespace fcpd

struct fcpd_ctx {
  // last spatial order of each point set, keyed on its normalised content
  // (repeated calls on the same clouds skip the k-d partition)
  struct SortCache {
    uint64_t hash = 0;
    int64_t count = -1;
    std::vector<int64_t> perm;
    std::vector<double> scratch;  // the gather's target, reused (no page faults per call)
  } sort_x, sort_y;
  // host staging of a register call, reused across calls: normalised points,
  // their float4 packing, the read-back (a fresh 5 MB vector per call costs
  // ~1 ms of page faults at C4)
  std::vector<double> host_xs, host_ys, host_xt, host_w;
  std::vector<float4> host_x4, host_y4;
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cublasHandle_t blas = nullptr;
  ncclComm_t comm = nullptr;  // set by fcpd_create_dist: scene-sharded EM over NCCL
  int rank = 0, world = 1;
  // scene-sharded sessions: the collective backend (NCCL: this rank; loopback:
  // every virtual rank) and, for a loopback group, its other ranks (owned)
  std::unique_ptr<fcpd::Comm> comm_obj;
  std::vector<fcpd_ctx*> loop_ranks;
  std::string err;
  fcpd::Basis basis;
  fcpd::Session sess;
};

namespace fcpd {
namespace {
// One rank per GPU (per process) over NCCL.
struct NcclComm : Comm {
  ncclComm_t c;
  NcclComm(ncclComm_t cc, int w) : c(cc) { world = w; }
  void reduce_scatter_sum(const std::vector<const double*>& send, const std::vector<double*>& recv,
                          size_t count, cudaStream_t s) override {
    FCPD_NCCL(ncclReduceScatter(send[0], recv[0], count, ncclDouble, ncclSum, c, s));
  }
  void all_reduce_sum(const std::vector<double*>& buf, size_t count, cudaStream_t s) override {
    FCPD_NCCL(ncclAllReduce(buf[0], buf[0], count, ncclDouble, ncclSum, c, s));
  }
  void all_reduce_max(const std::vector<float*>& buf, size_t count, cudaStream_t s) override {
    FCPD_NCCL(ncclAllReduce(buf[0], buf[0], count, ncclFloat, ncclMax, c, s));
  }
  void all_gather(const std::vector<const uint32_t*>& send, const std::vector<uint32_t*>& recv,
                  size_t words, cudaStream_t s) override {
    FCPD_NCCL(ncclAllGather(send[0], recv[0], words, ncclUint32, c, s));
  }
  void host_all_reduce(std::vector<std::vector<double>>& vals, bool max, cudaStream_t s) override {
    std::vector<double>& v = vals[0];
    double* d = nullptr;
    FCPD_CUDA(cudaMalloc(&d, sizeof(double) * std::max<size_t>(v.size(), 1)));
    FCPD_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, s));
    const ncclResult_t r = ncclAllReduce(d, d, v.size(), ncclDouble, max ? ncclMax : ncclSum, c, s);
    cudaMemcpyAsync(v.data(), d, sizeof(double) * v.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(d);
    if (r != ncclSuccess)
      throw Failure(FCPD_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  }
  // NCCL collectives are captured into the fallback's conditional node when
  // the runtime accepts it (session_begin_group re-captures unconditionally
  // otherwise)
  bool conditional_ok() const override { return true; }
};
}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FCPD_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

namespace {

int fail(fcpd_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <typename F>
int guarded(fcpd_ctx* ctx, F&& f) {
  if (!ctx) return FCPD_ERR_PARAMETER;
  try {
    FCPD_CUDA(cudaSetDevice(ctx->device));
    f();
    ctx->err.clear();
    return FCPD_OK;
  } catch (const Failure& e) {
    return fail(ctx, e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, FCPD_ERR_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, FCPD_ERR_CUDA, e.what());
  }
}

// pack a column-major M×D fp64 host point set into fp64 SoA(3) + float4
void pack_points(const double* src, int64_t cnt, int d, std::vector<double>& soa3,
                 std::vector<float4>& f4) {
  soa3.assign(3 * cnt, 0.0);
  f4.resize(cnt);
  for (int c = 0; c < d; ++c) std::memcpy(&soa3[c * cnt], src + c * cnt, sizeof(double) * cnt);
  for (int64_t i = 0; i < cnt; ++i)
    f4[i] = make_float4(static_cast<float>(soa3[i]), static_cast<float>(soa3[cnt + i]),
                        static_cast<float>(soa3[2 * cnt + i]), 0.f);
}

void validate_register(const double* x, int64_t m, const double* y, int64_t n, int d,
                       const fcpd_config& cfg) {
  // registration.hpp:82-86
  if (m <= 0 || n <= 0 || !x || !y) throw Failure(FCPD_ERR_PARAMETER, "register: empty point set");
  if (d < 1) throw Failure(FCPD_ERR_DIMENSION, "register: model and scene dimension mismatch");
  if (cfg.iterations < 0) throw Failure(FCPD_ERR_PARAMETER, "register: negative iterations");
  if (d > 3)
    throw Failure(FCPD_ERR_DIMENSION, "register: the B200 path supports D <= 3, got D=" +
                                          std::to_string(d));
  if (cfg.variant != FCPD_VARIANT_FAST && cfg.variant != FCPD_VARIANT_FAST_LOWRANK)
    throw Failure(FCPD_ERR_PARAMETER,
                  "register: only the fast / fast_lowrank variants run on the B200 path");
  if (m > INT32_MAX || n > INT32_MAX) throw Failure(FCPD_ERR_PARAMETER, "register: too many points");
  if (!(cfg.spectral_tau >= 0.0 && cfg.spectral_tau < 1.0))
    throw Failure(FCPD_ERR_PARAMETER, "register: spectral_tau must lie in [0, 1)");
}

int64_t lowrank_rank(double fraction, int64_t m) {  // solvers.hpp:46-54
  if (fraction <= 0.0 || fraction > 1.0)
    throw Failure(FCPD_ERR_PARAMETER, "rank_fraction must lie in (0, 1]");
  int64_t k = std::llround(fraction * static_cast<double>(m));
  return std::max<int64_t>(1, std::min<int64_t>(k, m));
}

constexpr int64_t kDenseEigLimit = 46000;          // M×M fp64 + syevd workspace fit
constexpr int64_t kDenseEigLimitLowrank = 16384;   // above: on-the-fly top-K solver
// power steps of the top-K subspace iteration, at most (FCPD_TOPK_ITERS
// overrides).  The solver stops early once every top-K Ritz residual is at
// 1e-11·θ₁ (topk.cu; FCPD_TOPK_ADAPTIVE=0 runs all steps): two steps reach
// the fp64 floor at full C2/C4 size but not the eigenpairs near rank K at
// small M (K/M = 2 %: eigenvalues off by 2e-10·λ₁, a top-K registration
// 2.7e-4 from the dense-basis one), which four meet
constexpr int kTopkIterations = 4;
int topk_iterations() {
  if (const char* e = std::getenv("FCPD_TOPK_ITERS")) return std::max(0, std::atoi(e));
  return kTopkIterations;
}
bool topk_adaptive() {
  const char* e = std::getenv("FCPD_TOPK_ADAPTIVE");
  return !(e && e[0] == '0');
}

void ensure_basis(fcpd_ctx* ctx, Session& s, const std::vector<double>& x_soa) {
  const bool lowrank = s.cfg.variant == FCPD_VARIANT_FAST_LOWRANK;
  const int64_t rank = lowrank ? lowrank_rank(s.cfg.rank_fraction, s.m) : s.m;
  if (!(s.cfg.beta > 0.0)) throw Failure(FCPD_ERR_PARAMETER, "build_gram: beta must be positive");
  uint64_t h = fnv1a(x_soa.data(), sizeof(double) * x_soa.size());
  h = fnv1a(&s.m, sizeof s.m, h);
  h = fnv1a(&rank, sizeof rank, h);
  Basis& b = ctx->basis;
  if (b.q && b.key_hash == h && b.key_beta == s.cfg.beta && b.m == s.m && b.k == rank &&
      b.key_variant == s.cfg.variant) {
    s.basis_reused = true;
    s.t_eig = 0.0;
    s.t_gram = 0.0;
    return;
  }
  s.basis_reused = false;
  b.release();
  // Low rank beyond the dense limit: top-K eigenpairs from on-the-fly Φ·V
  // products (topk.cu); Φ is never formed.  Small problems keep the
  // reference's full eigensolve + truncation exactly.
  // FCPD_TOPK_MIN_M overrides the switch-over point (tests force the top-K
  // path at small M to compare it with the dense solver)
  int64_t topk_min = kDenseEigLimitLowrank;
  if (const char* e = std::getenv("FCPD_TOPK_MIN_M")) topk_min = std::atoll(e);
  if (lowrank && s.m > topk_min) {
    const auto t1 = Clock::now();
    topk_eigensolve(ctx->solver, ctx->blas, s.x0.p, s.m, s.d, s.cfg.beta, rank,
                    topk_iterations(), topk_adaptive(), s.cfg.seed, b, ctx->stream);
    upload_lambda(b, false, ctx->stream);
    s.t_gram = 0.0;
    s.t_eig = since(t1);
    b.key_hash = h;
    b.key_beta = s.cfg.beta;
    b.key_variant = s.cfg.variant;
    b.t_gram = s.t_gram;
    b.t_eig = s.t_eig;
    return;
  }
  if (s.m > kDenseEigLimit)
    throw Failure(FCPD_ERR_PARAMETER,
                  "eigendecompose: the full-rank variant needs a dense M×M eigensolve; "
                  "M > " + std::to_string(kDenseEigLimit) + " — use fast_lowrank");
  double* phi = nullptr;
  FCPD_CUDA(cudaMalloc(&phi, sizeof(double) * s.m * s.m));
  try {
    const auto t0 = Clock::now();
    build_gram_device(s.x0.p, s.m, s.d, s.cfg.beta, phi, s.m, ctx->stream);
    FCPD_CUDA(cudaStreamSynchronize(ctx->stream));
    s.t_gram = since(t0);
    const auto t1 = Clock::now();
    dense_eigensolve(ctx->solver, phi, s.m, rank, b, nullptr, ctx->stream);
    upload_lambda(b, !lowrank, ctx->stream);
    s.t_eig = since(t1);
  } catch (...) {
    cudaFree(phi);
    throw;
  }
  cudaFree(phi);
  b.key_hash = h;
  b.key_beta = s.cfg.beta;
  b.key_variant = s.cfg.variant;
  b.t_gram = s.t_gram;
  b.t_eig = s.t_eig;
}

// Culling pays once there are enough tile pairs to skip: below ~1k pairs
// (e.g. C0, 8×8 tiles) its four geometry kernels cost more than they save.
// FCPD_CULL=0/1 overrides.
constexpr int64_t kCullMinTilePairs = 1024;
bool cull_default(int64_t x_tiles, int64_t y_tiles) {
  if (const char* e = std::getenv("FCPD_CULL")) return std::atoi(e) != 0;
  return x_tiles * y_tiles >= kCullMinTilePairs;
}

// Wire the session's culling geometry into the E-step buffers.  margin =
// kCullMarginBits + log2(count) log2-units: the skipped mass is ≤ 2^-bits of
// any column/row total.  32 bits (2.3e-10 relative) sits far below the fp32
// pair terms' own rounding (≈ |t|·2^-24 per term) and the 1e-5 σ² parity
// bar; FCPD_CULL_MARGIN overrides.
constexpr float kCullMarginBits = 32.f;
float cull_margin_bits() {
  if (const char* e = std::getenv("FCPD_CULL_MARGIN")) return static_cast<float>(std::atof(e));
  return kCullMarginBits;
}

void set_cull(Session& s, EStepBuffers& eb, int64_t m, int64_t n_local, int64_t n_global) {
  CullInfo& c = eb.cull;
  c.enabled = s.cull && s.xlo.p && s.ylo.p && s.wl1_tiles.p && s.wl2_tiles.p ? 1 : 0;
  const char* pe = std::getenv("FCPD_CULL_PROBE");
  c.probe = pe ? (std::atoi(pe) != 0) : 1;
  c.n_xtiles = ceil_div(m, kTilePts);
  c.n_ytiles = ceil_div(n_local, kTilePts);
  c.n_xsub = ceil_div(m, kSubPts);
  c.n_ysub = ceil_div(n_local, kSubPts);
  c.xlo = s.xlo.p;
  c.xhi = s.xhi.p;
  c.ylo = s.ylo.p;
  c.yhi = s.yhi.p;
  c.bminmax = s.bminmax.p;
  c.sxlo = s.sxlo.p;
  c.sxhi = s.sxhi.p;
  c.sylo = s.sylo.p;
  c.syhi = s.syhi.p;
  c.sbminmax = s.sbminmax.p;
  const float bits = cull_margin_bits();
  c.margin1 = bits + static_cast<float>(std::log2(static_cast<double>(std::max<int64_t>(m, 1))));
  c.margin2 =
      bits + static_cast<float>(std::log2(static_cast<double>(std::max<int64_t>(n_global, 1))));
  c.counters = s.cull_counters.p;
  c.wl1_offset = s.wl1_off.p;
  c.wl1_units = static_cast<int64_t>(c.n_ytiles) * c.n_xsub;
  c.wl2_units = static_cast<int64_t>(c.n_xtiles) * c.n_ysub;
  c.probe_paid1 = s.probe_paid.p;
  c.probe_paid2 = s.probe_paid.p ? s.probe_paid.p + c.n_ytiles : nullptr;
  eb.cullw = CullBuffers{s.xlo.p,  s.xhi.p,  s.ylo.p,  s.yhi.p,  s.bminmax.p,
                         s.sxlo.p, s.sxhi.p, s.sylo.p, s.syhi.p, s.sbminmax.p};
  eb.wl1 = WorkListBuffers{s.wl1_tiles.p, s.wl1_off.p, s.wl_done.p};
  eb.wl2 = WorkListBuffers{s.wl2_tiles.p, s.wl2_off.p, s.wl_done.p ? s.wl_done.p + 1 : nullptr};
}

// E-step buffers of the session (pt1: optional Σ_m P_mn output; resid:
// write R = P̃Y − X for the M-step; row_aos: distributed row sums instead).
EStepBuffers estep_buffers(Session& s, double* pt1, bool resid, double* row_aos = nullptr) {
  EStepBuffers eb{};
  eb.xt4 = s.xt4.p;
  eb.xt64 = s.xt64.p;
  eb.y4b = s.y4b.p;
  eb.b2 = s.b2.p;
  eb.pt1 = pt1;
  eb.col_seg = s.col_seg.p;
  eb.row_seg = s.row_seg.p;
  eb.col_done = s.col_done.p;
  eb.row_done = s.row_done.p;
  eb.col_flags = s.col_flags.p;
  eb.row_flags = s.row_flags.p;
  eb.out = RowOut{s.ptilde_y.p, s.var.p, s.log2p1.p, s.degenerate.p,
                  resid ? s.resid4.p : nullptr, resid ? s.x0.p : nullptr};
  eb.ystats = s.ystats;
  eb.row_aos = row_aos;
  eb.stamps = s.stamps.p;
  set_cull(s, eb, s.m, s.n, s.dist ? s.n_global : s.n);
  return eb;
}

// Session E-step scratch: segment partials, work lists, culling geometry.
// m = model rows the E-step sees (all M), n = local scene points.
void alloc_estep(Session& s, int64_t m, int64_t n, cudaStream_t str) {
  s.col_seg.ensure(s.ep.col_seg_doubles());
  s.row_seg.ensure(s.ep.row_seg_doubles());
  // block arrival counters of the pass fix-ups (self-resetting)
  s.col_done.ensure(s.ep.col_blocks);
  s.row_done.ensure(s.ep.row_blocks);
  FCPD_CUDA(cudaMemsetAsync(s.col_done.p, 0, sizeof(int32_t) * s.ep.col_blocks, str));
  FCPD_CUDA(cudaMemsetAsync(s.row_done.p, 0, sizeof(int32_t) * s.ep.row_blocks, str));
  const int64_t nxt = ceil_div(m, kTilePts), nyt = ceil_div(n, kTilePts);
  const int64_t nxs = ceil_div(m, kSubPts), nys = ceil_div(n, kSubPts);
  s.cull = cull_default(nxt, nyt);
  s.xlo.ensure(nxt);
  s.xhi.ensure(nxt);
  s.ylo.ensure(nyt);
  s.yhi.ensure(nyt);
  s.bminmax.ensure(nyt);
  s.sxlo.ensure(nxs);
  s.sxhi.ensure(nxs);
  s.sylo.ensure(nys);
  s.syhi.ensure(nys);
  s.sbminmax.ensure(nys);
  // [0..1] (block, sub-tile) units evaluated per pass, [2..5] pair slots by
  // (pass, form) — cumulative over the session
  s.cull_counters.ensure(6);
  FCPD_CUDA(cudaMemsetAsync(s.cull_counters.p, 0, 6 * sizeof(unsigned long long), str));
  s.probe_paid.ensure(nxt + nyt);
  FCPD_CUDA(cudaMemsetAsync(s.probe_paid.p, 1, (nxt + nyt) * sizeof(int32_t), str));  // ≠ 0
  if (s.cull) {
    s.wl1_tiles.ensure(static_cast<size_t>(nyt) * nxs);
    s.wl1_off.ensure(nyt + 1);
    s.wl2_tiles.ensure(static_cast<size_t>(nxt) * nys);
    s.wl2_off.ensure(nxt + 1);
    s.wl_done.ensure(2);
    FCPD_CUDA(cudaMemsetAsync(s.wl_done.p, 0, 2 * sizeof(int32_t), str));
  }
  launch_tile_bbox(s.y4b.p, n, s.ylo.p, s.yhi.p, s.sylo.p, s.syhi.p, nullptr, str);
}

// ev (optional, 7 events): recorded before the iteration and after each of
// pass 1, pass 2, Qᵀ·R, z-reduce/filter, Q·g, transform/σ² (eager profiling).
void enqueue_iteration(fcpd_ctx* ctx, Session& s, cudaEvent_t* ev = nullptr) {
  Basis& b = ctx->basis;
  IterState* st = s.st.p;
  cudaStream_t str = ctx->stream;
  const EStepBuffers eb = estep_buffers(s, nullptr, true);
  auto rec = [&](int i) {
    if (ev) FCPD_CUDA(cudaEventRecord(ev[i], str));
  };
  rec(0);
  const MstepFusedArgs fa{b.q, b.kpad, b.k, b.lam, b.lam + b.k, s.cfg.lambda_reg, s.tau,
                          s.zp.trunc, s.resid4.p, s.zpart_fused.p, s.coef.p, s.g4.p, s.x0.p,
                          s.xt64.p, s.xt_prev.p, s.xt4.p, s.ptilde_y.p, s.var.p, s.sig_part.p,
                          s.mfused_done.p, s.m, s.d, s.cfg.early_stop, s.trace.p, st,
                          s.stamps.p};
  if (s.small) {  // the whole iteration as one cooperative kernel (booked as the E-step)
    const SmallIterArgs sa{fa, s.y4b.p, s.b2.p, s.n, eb.out, eb.ystats, s.cull_counters.p};
    launch_small_iter(sa, s.mfused_grid, str);
    for (int i = 1; i <= 6; ++i) rec(i);
    return;
  }
  launch_estep(s.ep, eb, s.m, s.n, st, str, ev ? ev[1] : nullptr);
  rec(2);
  if (s.mfused) {  // one cooperative kernel; its time is booked as the Qᵀ·R phase
    launch_mstep_fused(fa, s.mfused_grid, str);
    for (int i = 3; i <= 6; ++i) rec(i);
    return;
  }
  if (s.zp.trunc)
    launch_spectral_rank(b.lam, b.lam + b.k, b.k, s.cfg.lambda_reg, s.tau, st, str);
  if (s.rowdot) {
    launch_rowdot(s.zr, b.qt, s.resid4.p, s.zpart.p, st, s.stamps.p, 1, str);
    rec(3);
    launch_rowdot_reduce(s.zr, s.zpart.p, b.k, b.lam, b.lam + b.k, s.cfg.lambda_reg, s.coef.p,
                         s.g4.p, nullptr, st, str);
  } else {
    launch_colsum(s.zp, b.q, b.kpad, s.resid4.p, s.zpart.p, st, s.stamps.p, 1, str);
    rec(3);
    launch_zreduce(s.zp, s.zpart.p, b.lam, b.lam + b.k, s.cfg.lambda_reg, s.coef.p, s.g4.p, st,
                   str);
  }
  rec(4);
  launch_colsum(s.vp, b.qt, b.mpad, s.g4.p, s.vpart.p, st, nullptr, 0, str);
  rec(5);
  launch_transform_sigma(s.vp, s.vpart.p, s.x0.p, s.xt64.p, s.xt_prev.p, s.xt4.p, s.ptilde_y.p,
                         s.var.p, s.sig_part.p, s.d, s.cfg.early_stop, s.trace.p, st,
                         s.stamps.p, str);
  rec(6);
}

}  // namespace
}  // namespace fcpd

namespace fcpd {
namespace {

// Upload points, plan kernels, allocate per-session device buffers.
// x_soa/y_soa are fp64 SoA(3) host arrays already normalised.
void prepare_buffers(fcpd_ctx* ctx, Session& s, const std::vector<double>& x_soa,
                     const std::vector<double>& y_soa, int capacity, bool need_mstep,
                     bool x0_on_device = false) {
  const int64_t m = s.m, n = s.n;
  cudaStream_t str = ctx->stream;
  s.x0.ensure(3 * m);
  s.xt64.ensure(3 * m);
  s.xt_prev.ensure(3 * m);
  s.y64.ensure(3 * n);
  s.xt4.ensure(m);
  s.y4b.ensure(n);
  s.resid4.ensure(m);
  s.b2.ensure(n);
  s.pt1.ensure(n);
  s.ptilde_y.ensure(3 * m);
  s.var.ensure(m);
  s.log2p1.ensure(m);
  s.degenerate.ensure(m);
  s.col_flags.ensure(n);
  s.row_flags.ensure(m);
  s.st.ensure(1);
  s.capacity = std::max(capacity, 1);
  s.trace.ensure(s.capacity);
  s.stamps.ensure(4 * static_cast<size_t>(s.capacity));
  s.ep = make_estep_plan(m, n, ctx->sm_count);
  s.sig_part.ensure(transform_sigma_blocks(m));  // one σ² partial per transform block

  std::vector<float4>& x4 = ctx->host_x4;
  std::vector<float4>& y4 = ctx->host_y4;
  x4.resize(m);
  y4.resize(n);
  YStats ys{};
  parallel_for(m + n >= 65536 ? 2 : 1, [&](int t) {
    for (int k = t; k < 2; k += (m + n >= 65536 ? 2 : 1)) {
      if (k == 0) {
        for (int64_t i = 0; i < m; ++i)
          x4[i] = make_float4(static_cast<float>(x_soa[i]), static_cast<float>(x_soa[m + i]),
                              static_cast<float>(x_soa[2 * m + i]), 0.f);
      } else {
        for (int64_t i = 0; i < n; ++i)
          y4[i] = make_float4(static_cast<float>(y_soa[i]), static_cast<float>(y_soa[n + i]),
                              static_cast<float>(y_soa[2 * n + i]), 0.f);
        // scene statistics for the uniform-row fallback (fp64, fixed order)
        for (int c = 0; c < 3; ++c) {
          double acc = 0.0;
          for (int64_t i = 0; i < n; ++i) acc += y_soa[c * n + i];
          ys.mean[c] = acc / static_cast<double>(n);
        }
        double sq = 0.0;
        for (int64_t i = 0; i < n; ++i)
          sq += y_soa[i] * y_soa[i] + y_soa[n + i] * y_soa[n + i] + y_soa[2 * n + i] * y_soa[2 * n + i];
        ys.sq_mean = sq / static_cast<double>(n);
      }
    }
  });
  if (!x0_on_device)  // (session_begin uploads X before the basis build)
    FCPD_CUDA(cudaMemcpyAsync(s.x0.p, x_soa.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.xt64.p, s.x0.p, sizeof(double) * 3 * m, cudaMemcpyDeviceToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.xt_prev.p, s.x0.p, sizeof(double) * 3 * m, cudaMemcpyDeviceToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.y64.p, y_soa.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.xt4.p, x4.data(), sizeof(float4) * m, cudaMemcpyHostToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.y4b.p, y4.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, str));
  s.h2d += (sizeof(double) * 3 + sizeof(float4)) * (m + n);

  s.ystats = ys;

  alloc_estep(s, m, n, str);  // scene tiles are fixed for the session

  if (need_mstep) {
    Basis& b = ctx->basis;
    s.zp = make_colsum_plan(m, b.k, ctx->sm_count);
    s.vp = make_colsum_plan(b.k, m, ctx->sm_count);
    // The fused M-step pays where the streamed basis is small enough that
    // the two passes are latency-bound and its re-read of Q hits L2: a basis
    // ≤ 64 MB, or a truncated one over M ≤ 32k rows (FCPD_MSTEP_FUSED=0/1).
    const double qbytes = 4.0 * static_cast<double>(m) * static_cast<double>(b.k);
    s.mfused = qbytes <= 64.0 * (1 << 20) || (s.cfg.spectral_tau > 0.0 && m <= 32768);
    if (const char* e = std::getenv("FCPD_MSTEP_FUSED")) s.mfused = std::atoi(e) != 0;
    // spectral truncation: the basis streams stop where the filter drops
    // below tau (mstep.cu: spectral_rank_kernel; phase 0 of the fused
    // kernel).  A basis under 64 MB on the streaming path streams in
    // microseconds, so there its extra kernel would cost more than it saves;
    // the fused kernel's search is free (C0: 13.4k → 15.2k it/s).
    // FCPD_SPECTRAL_TAU=0 → off
    s.tau = s.cfg.spectral_tau;
    if (!s.mfused && qbytes < 64.0 * (1 << 20)) s.tau = 0.0;
    if (const char* e = std::getenv("FCPD_SPECTRAL_TAU")) s.tau = std::atof(e);  // A/B
    s.zp.trunc = s.tau > 0.0 ? 1 : 0;
    s.vp.trunc = s.tau > 0.0 ? 2 : 0;
    const char* zpass = std::getenv("FCPD_ZPASS");
    s.rowdot = !s.mfused && !(zpass && std::string(zpass) == "colsum");
    s.zr = make_rowdot_plan(b.k, m, b.mpad, ctx->sm_count);
    s.zr.g.trunc = s.zp.trunc;
    s.zpart.ensure(std::max(s.zp.part_doubles(), s.rowdot ? s.zr.part_doubles() : size_t(0)));
    s.vpart.ensure(s.vp.part_doubles());
    s.coef.ensure(3 * b.k);
    s.g4.ensure(b.kpad);  // the fused M-step streams whole quads (kpad ≥ K)
    if (s.mfused) {
      s.mfused_grid = mstep_fused_grid(ctx->sm_count);
      s.zpart_fused.ensure(static_cast<size_t>(b.k) * s.mfused_grid * 3);
      s.mfused_done.ensure(1);
      FCPD_CUDA(cudaMemsetAsync(s.mfused_done.p, 0, sizeof(int32_t), str));
      s.sig_part.ensure(std::max(transform_sigma_blocks(m), s.mfused_grid));
    }
    // small problems: the whole iteration as one kernel (FCPD_SMALL_ITER=0/1)
    s.small = !s.dist && s.mfused && !s.cull && small_iter_fits(m, s.n);
    if (const char* e = std::getenv("FCPD_SMALL_ITER"))
      s.small = std::atoi(e) != 0 && !s.dist && s.mfused && !s.cull && small_iter_fits(m, s.n);
  }
}

// Iteration-0 state: σ², then the E-step scalars on the device (the code
// every later iteration uses for its σ²); ω, M, global N, D.
void reset_state(fcpd_ctx* ctx, Session& s, double sigma2) {
  IterState h{};
  h.sigma2 = sigma2;
  h.sigma2_e = sigma2;
  h.active = 1;
  FCPD_CUDA(cudaMemcpyAsync(s.st.p, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
  launch_init_state(s.st.p, sigma2, s.cfg.omega, s.m, s.dist ? s.n_global : s.n, s.d,
                    ctx->stream);
  FCPD_CUDA(cudaMemsetAsync(s.degenerate.p, 0, sizeof(int32_t) * (s.dist ? s.mr : s.m),
                            ctx->stream));
}

// registration.hpp:59-69 (host, fp64, same formula)
double init_sigma2_host(const std::vector<double>& x, int64_t m, const std::vector<double>& y,
                        int64_t n, int d) {
  double fx = 0.0, fy = 0.0, dot = 0.0;
  for (int c = 0; c < d; ++c) {
    double sx = 0.0, sy = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      fx += x[c * m + i] * x[c * m + i];
      sx += x[c * m + i];
    }
    for (int64_t i = 0; i < n; ++i) {
      fy += y[c * n + i] * y[c * n + i];
      sy += y[c * n + i];
    }
    dot += sx * sy;
  }
  const double md = static_cast<double>(m), nd = static_cast<double>(n);
  return std::max((md * fy + nd * fx - 2.0 * dot) / (static_cast<double>(d) * md * nd), 0.0);
}

void session_begin_dist(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n,
                        int d, const fcpd_config& cfg);
void session_read_dist(fcpd_ctx* ctx, fcpd_result* out, double wall);

// ---- spatial sort: makes every 256-point tile a compact box for the
// E-step's tile culling and its centred pair form.  A k-d partition: split
// the points at a multiple of 256 along the longest axis of their bounding
// box, recursively, so every tile is one leaf with a bounded aspect ratio,
// then each tile the same way at multiples of 32 (the culling sub-tiles)
// (a Morton order lets some tiles straddle distant cells, and those tiles
// lose both culling and the centred form).  Depth-first leaf order keeps
// consecutive tiles near each other.  The order depends only on the point
// set, is deterministic (ties by index), and is undone on every output.
namespace {
void kd_partition(const std::vector<double>& soa, int64_t cnt, int64_t* idx, int64_t len,
                  int par_depth = 2, int64_t kLeaf = kTilePts) {
  if (len <= kLeaf) {  // a tile: split it the same way into 32-point sub-tiles
    if (kLeaf == kTilePts && len > kSubPts) kd_partition(soa, cnt, idx, len, 0, kSubPts);
    return;
  }
  while (len > kLeaf) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t k = 0; k < len; ++k)
      for (int c = 0; c < 3; ++c) {
        const double v = soa[c * cnt + idx[k]];
        lo[c] = std::min(lo[c], v);
        hi[c] = std::max(hi[c], v);
      }
    int axis = 0;
    for (int c = 1; c < 3; ++c)
      if (hi[c] - lo[c] > hi[axis] - lo[axis]) axis = c;
    const int64_t leaves = (len + kLeaf - 1) / kLeaf;
    const int64_t left = (leaves + 1) / 2 * kLeaf;  // a whole number of tiles
    const double* key = soa.data() + axis * cnt;
    std::nth_element(idx, idx + left, idx + len, [key](int64_t a, int64_t b) {
      return key[a] < key[b] || (key[a] == key[b] && a < b);
    });
    if (par_depth > 0 && len >= (int64_t(1) << 15)) {  // halves on separate threads
      std::thread t([&soa, cnt, idx, left, par_depth, kLeaf] {
        kd_partition(soa, cnt, idx, left, par_depth - 1, kLeaf);
      });
      kd_partition(soa, cnt, idx + left, len - left, par_depth - 1, kLeaf);
      t.join();
      return;
    }
    kd_partition(soa, cnt, idx, left, 0, kLeaf);
    idx += left;
    len -= left;
  }
  if (kLeaf == kTilePts && len > kSubPts) kd_partition(soa, cnt, idx, len, 0, kSubPts);
}
}  // namespace

// perm[k] = original index of sorted position k; soa (SoA 3×cnt) is permuted.
std::vector<int64_t> spatial_sort(std::vector<double>& soa, int64_t cnt) {
  std::vector<int64_t> perm(cnt);
  for (int64_t i = 0; i < cnt; ++i) perm[i] = i;
  kd_partition(soa, cnt, perm.data(), cnt);
  std::vector<double> out(soa.size());
  for (int c = 0; c < 3; ++c)
    for (int64_t k = 0; k < cnt; ++k) out[c * cnt + k] = soa[c * cnt + perm[k]];
  soa.swap(out);
  return perm;
}

// spatial_sort through a content-keyed cache: a hit applies the cached
// permutation (the same deterministic order the partition would produce).
template <typename Cache>
std::vector<int64_t> spatial_sort_cached(std::vector<double>& soa, int64_t cnt, Cache& c) {
  const uint64_t h = fnv1a(soa.data(), sizeof(double) * soa.size());
  if (c.count == cnt && c.hash == h && static_cast<int64_t>(c.perm.size()) == cnt) {
    std::vector<double>& out = c.scratch;
    out.resize(soa.size());
    parallel_for(cnt >= 65536 ? 3 : 1, [&](int t) {
      for (int d = t; d < 3; d += (cnt >= 65536 ? 3 : 1))
        for (int64_t k = 0; k < cnt; ++k) out[d * cnt + k] = soa[d * cnt + c.perm[k]];
    });
    soa.swap(out);
    return c.perm;
  }
  std::vector<int64_t> perm = spatial_sort(soa, cnt);
  c.hash = h;
  c.count = cnt;
  c.perm = perm;
  return perm;
}

// normalize_pair (pointset.hpp:124-148), fp64 on the host, O(M+N); outputs
// fp64 SoA(3) copies (unused coordinates zero).
void normalize_pair_host(const double* x, int64_t m, const double* y, int64_t n, int d,
                         bool normalize, std::vector<double>& xs, std::vector<double>& ys,
                         double* center, double* scale) {
  xs.assign(3 * m, 0.0);
  ys.assign(3 * n, 0.0);
  center[0] = center[1] = center[2] = 0.0;
  *scale = 1.0;
  if (normalize) {
    // one task per (coordinate, point set); each sum / max / write runs in
    // the serial order, so the result does not depend on the threading
    const int tasks = (m + n) >= 65536 ? 2 * d : 1;
    const double total = static_cast<double>(m + n);
    double part[6] = {0, 0, 0, 0, 0, 0};
    auto slice = [&](int t, auto&& body) {
      for (int k = t; k < 2 * d; k += tasks) {
        const int c = k >> 1;
        const bool is_y = k & 1;
        body(k, c, is_y ? y + c * n : x + c * m, is_y ? n : m, is_y ? &ys[c * n] : &xs[c * m]);
      }
    };
    parallel_for(tasks, [&](int t) {
      slice(t, [&](int k, int, const double* src, int64_t cnt, double*) {
        double acc = 0.0;
        for (int64_t i = 0; i < cnt; ++i) acc += src[i];
        part[k] = acc;
      });
    });
    for (int c = 0; c < d; ++c) center[c] = (part[2 * c] + part[2 * c + 1]) / total;
    parallel_for(tasks, [&](int t) {
      slice(t, [&](int k, int c, const double* src, int64_t cnt, double*) {
        double mx = 0.0;
        for (int64_t i = 0; i < cnt; ++i) mx = std::max(mx, std::fabs(src[i] - center[c]));
        part[k] = mx;
      });
    });
    double sc = 0.0;
    for (int k = 0; k < 2 * d; ++k) sc = std::max(sc, part[k]);
    if (sc <= 0.0) sc = 1.0;
    *scale = sc;
    parallel_for(tasks, [&](int t) {
      slice(t, [&](int, int c, const double* src, int64_t cnt, double* dst) {
        for (int64_t i = 0; i < cnt; ++i) dst[i] = (src[i] - center[c]) / sc;
      });
    });
  } else {
    for (int c = 0; c < d; ++c) {
      std::memcpy(&xs[c * m], x + c * m, sizeof(double) * m);
      std::memcpy(&ys[c * n], y + c * n, sizeof(double) * n);
    }
  }
}

void session_begin(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n, int d,
                   const fcpd_config& cfg) {
  if (ctx->comm_obj) {
    session_begin_dist(ctx, x, m, y, n, d, cfg);
    return;
  }
  validate_register(x, m, y, n, d, cfg);
  const auto t0 = Clock::now();
  Session& s = ctx->sess;
  s.ready = false;
  s.dist = false;
  s.h2d = s.d2h = 0;
  s.m = m;
  s.n = n;
  s.d = d;
  s.cfg = cfg;
  static const bool host_timing = std::getenv("FCPD_HOST_TIMING") != nullptr;
  auto stamp = [&](const char* what) {
    if (host_timing) std::fprintf(stderr, "[fcpd] begin %-12s %8.3f ms\n", what, 1e3 * since(t0));
  };
  std::vector<double>& xs = ctx->host_xs;
  std::vector<double>& ys = ctx->host_ys;
  normalize_pair_host(x, m, y, n, d, cfg.normalize != 0, xs, ys, s.center, &s.scale);
  stamp("normalize");
  // internal order: spatially sorted model and scene (undone on output); the
  // two sorts are independent
  {
    std::thread tx([&] { s.perm_x = spatial_sort_cached(xs, m, ctx->sort_x); });
    s.perm_y = spatial_sort_cached(ys, n, ctx->sort_y);
    tx.join();
  }
  stamp("spatial_sort");
  // x0 must be on the device before the Gram build
  s.x0.ensure(3 * m);
  FCPD_CUDA(cudaMemcpyAsync(s.x0.p, xs.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice,
                            ctx->stream));
  ensure_basis(ctx, s, xs);
  stamp("basis");
  ctx->basis.perm = s.perm_x;  // basis rows are in the session's sorted order
  prepare_buffers(ctx, s, xs, ys, cfg.iterations, true, /*x0_on_device=*/true);
  stamp("buffers");
  s.sigma2_initial = init_sigma2_host(xs, m, ys, n, d);
  if (cfg.iterations > 0 && !(cfg.omega >= 0.0 && cfg.omega < 1.0))
    throw Failure(FCPD_ERR_NUMERIC,
                  "register: iteration 0: posterior: omega must lie in [0, 1)");
  reset_state(ctx, s, s.sigma2_initial);
  FCPD_CUDA(cudaMemsetAsync(s.coef.p, 0, sizeof(double) * 3 * ctx->basis.k, ctx->stream));

  stamp("state");
  // capture one EM iteration as a CUDA graph
  cudaGraph_t g = nullptr;
  FCPD_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_iteration(ctx, s);
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  FCPD_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  // a repeated register call with the same shapes captures the same graph
  // topology: update the existing executable instead of re-instantiating
  bool updated = false;
  if (s.graph) {
    cudaGraphExecUpdateResultInfo info{};
    updated = cudaGraphExecUpdate(s.graph, g, &info) == cudaSuccess;
    if (!updated) {
      cudaGetLastError();  // clear the update failure
      s.release_graph();
    }
  }
  if (!updated) {
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    FCPD_CUDA(ie);
    s.graph = exec;
  } else {
    cudaGraphDestroy(g);
  }
  stamp("graph");
  FCPD_CUDA(cudaStreamSynchronize(ctx->stream));
  stamp("sync");
  s.t_setup_host = since(t0);
  s.launched = 0;
  s.ready = true;
}

void session_run(fcpd_ctx* ctx, int iters) {
  Session& s = ctx->sess;
  if (!s.ready) throw Failure(FCPD_ERR_PARAMETER, "session: not started");
  if (iters < 0 || s.launched + iters > s.capacity)
    throw Failure(FCPD_ERR_PARAMETER, "session: more iterations than cfg.iterations");
  s.launched += iters;
  for (int i = 0; i < iters; ++i) FCPD_CUDA(cudaGraphLaunch(s.graph, ctx->stream));
}

void session_read(fcpd_ctx* ctx, fcpd_result* out, double wall) {
  if (ctx->sess.dist) {
    session_read_dist(ctx, out, wall);
    return;
  }
  Session& s = ctx->sess;
  Basis& b = ctx->basis;
  cudaStream_t str = ctx->stream;
  IterState h{};
  FCPD_CUDA(cudaMemcpyAsync(&h, s.st.p, sizeof h, cudaMemcpyDeviceToHost, str));
  FCPD_CUDA(cudaStreamSynchronize(str));
  s.d2h += sizeof h;
  if (h.err_code != 0) {
    std::string what;
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", h.err_value);
    if (h.err_code == kDevSolveDiag) what = "solve_fast: lambda_i + lambda*sigma2 not positive";
    else what = std::string("update_sigma2: negative variance ") + buf;
    throw Failure(FCPD_ERR_NUMERIC, "register: iteration " + std::to_string(h.err_iter) + ": " + what);
  }
  const int64_t m = s.m, n = s.n;
  const int d = s.d;
  const int run = h.iters_run;
  if (!out) return;
  out->iterations_run = run;
  out->basis_reused = s.basis_reused ? 1 : 0;
  out->sigma2_initial = s.sigma2_initial;
  out->degenerate_rows = h.degenerate_rows;
  out->sigma2_clamps = h.sigma2_clamps;
  if (out->sigma2_trace && run > 0)
    FCPD_CUDA(cudaMemcpyAsync(out->sigma2_trace, s.trace.p, sizeof(double) * run,
                              cudaMemcpyDeviceToHost, str));
  s.d2h += sizeof(double) * (run + 3 * m);
  std::vector<double>& xt = ctx->host_xt;
  xt.resize(3 * m);
  FCPD_CUDA(cudaMemcpyAsync(xt.data(), s.xt64.p, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, str));
  // internal rows are spatially sorted: sorted row k is original row perm_x[k]
  const std::vector<int64_t>& px = s.perm_x;
  const std::vector<int64_t>& py = s.perm_y;
  if (out->coefficients) {
    // W = Q c (the last iteration's coefficients).  With a truncated basis
    // stream the iterations only formed c for the kept eigenpairs: redo z
    // over the full basis from the last residual, then one Qᵀ-row stream.
    if (s.zp.trunc && run > 0) {
      launch_colsum(s.zp, b.q, b.kpad, s.resid4.p, s.zpart.p, nullptr, nullptr, 0, str);
      launch_zcoef(s.zp, s.zpart.p, b.lam, s.cfg.lambda_reg, s.coef.p, s.st.p, str);
    }
    pack_coef_kernel<<<ceil_div(b.k, 256), 256, 0, str>>>(s.coef.p, b.k, s.g4.p);
    FCPD_LAUNCH_CHECK();
    launch_colsum(s.vp, b.qt, b.mpad, s.g4.p, s.vpart.p, nullptr, nullptr, 0, str);
    launch_vreduce_add(s.vp, s.vpart.p, nullptr, d, s.ptilde_y.p, str);
    std::vector<double>& w = ctx->host_w;
    w.resize(static_cast<size_t>(d) * m);
    FCPD_CUDA(cudaMemcpyAsync(w.data(), s.ptilde_y.p, sizeof(double) * d * m,
                              cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaStreamSynchronize(str));
    parallel_for(m >= 65536 ? d : 1, [&](int t) {
      for (int c = t; c < d; c += (m >= 65536 ? d : 1))
        for (int64_t k = 0; k < m; ++k) out->coefficients[c * m + px[k]] = w[c * m + k];
    });
    s.d2h += sizeof(double) * d * m;
  }
  if (out->correspondence && run > 0) {
    DevBuf<double> p;
    p.ensure(static_cast<size_t>(m) * n);
    // the last E-step's P̃ (x̃ before the last transform, σ² it used)
    DevBuf<int32_t> deg;
    deg.ensure(m);
    launch_dense_posterior(s.xt_prev.p, m, s.y64.p, n, d, s.cfg.omega, s.st.p, 1, deg.p, p.p,
                           str);
    std::vector<double> ps(static_cast<size_t>(m) * n);
    FCPD_CUDA(cudaMemcpyAsync(ps.data(), p.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost,
                              str));
    s.d2h += sizeof(double) * m * n;
    FCPD_CUDA(cudaStreamSynchronize(str));
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = 0; k < m; ++k) out->correspondence[py[j] * m + px[k]] = ps[j * m + k];
    p.release();
    deg.release();
  }
  std::vector<int32_t> degm(out->degenerate_mask ? m : 0);
  if (out->degenerate_mask) {
    FCPD_CUDA(cudaMemcpyAsync(degm.data(), s.degenerate.p, sizeof(int32_t) * m,
                              cudaMemcpyDeviceToHost, str));
    s.d2h += sizeof(int32_t) * m;
  }
  std::vector<uint64_t> stamps(4 * static_cast<size_t>(std::max(run, 1)));
  if (run > 0)
    FCPD_CUDA(cudaMemcpyAsync(stamps.data(), s.stamps.p, sizeof(uint64_t) * 4 * run,
                              cudaMemcpyDeviceToHost, str));
  s.d2h += sizeof(uint64_t) * 4 * run;
  unsigned long long tiles[6] = {0, 0, 0, 0, 0, 0};
  if (s.cull_counters.p)
    FCPD_CUDA(cudaMemcpyAsync(tiles, s.cull_counters.p, sizeof tiles, cudaMemcpyDeviceToHost, str));
  FCPD_CUDA(cudaStreamSynchronize(str));
  out->tiles_evaluated[0] = static_cast<int64_t>(tiles[0]);
  out->tiles_evaluated[1] = static_cast<int64_t>(tiles[1]);
  for (int k = 0; k < 4; ++k) out->pairs_by_form[k] = static_cast<int64_t>(tiles[2 + k]);
  out->spectral_rank = s.zp.trunc && h.keff > 0 ? std::min<int64_t>(h.keff, b.k) : b.k;
  out->mstep_fused = s.mfused ? 1 : 0;
  if (out->degenerate_mask)
    for (int64_t k = 0; k < m; ++k) out->degenerate_mask[px[k]] = degm[k];
  if (out->transformed) {
    parallel_for(m >= 65536 ? d : 1, [&](int t) {
      for (int c = t; c < d; c += (m >= 65536 ? d : 1))
        for (int64_t k = 0; k < m; ++k)
          out->transformed[c * m + px[k]] =
              s.cfg.normalize ? xt[c * m + k] * s.scale + s.center[c] : xt[c * m + k];
    });
  }
  // phases (registration.hpp:120-147): t_c = E-step; t_iter = residual +
  // solve (Qᵀ R, filter, Q g); t_o = transform epilogue + σ² + everything else
  double tc = 0.0, ti = 0.0;
  for (int it = 0; it < run; ++it) {
    const uint64_t* st4 = &stamps[4 * it];
    tc += 1e-9 * static_cast<double>(st4[1] - st4[0]);
    ti += 1e-9 * static_cast<double>(st4[2] - st4[1]);
  }
  if (std::getenv("FCPD_HOST_TIMING") && run > 1) {  // device phase split (diagnostic)
    double t3 = 0.0, gap = 0.0;
    for (int it = 0; it < run; ++it) t3 += 1e-9 * static_cast<double>(stamps[4 * it + 3] - stamps[4 * it + 2]);
    for (int it = 0; it + 1 < run; ++it)
      gap += 1e-9 * static_cast<double>(stamps[4 * (it + 1)] - stamps[4 * it + 3]);
    std::fprintf(stderr,
                 "[fcpd] per iteration: E-step %.2f us, M-step to V %.2f us, transform+σ² %.2f us, "
                 "gap to next %.2f us\n",
                 1e6 * tc / run, 1e6 * ti / run, 1e6 * t3 / run, 1e6 * gap / (run - 1));
  }
  fcpd_timing& t = out->timing;
  t.t_c = tc;
  t.t_eig = s.t_eig;
  t.t_iter = ti;
  t.t_f = t.t_eig + t.t_iter;
  t.t_o = std::max(wall - t.t_c - t.t_f, 0.0);
  t.t_total = t.t_c + t.t_f + t.t_o;
  t.t_setup = s.t_gram + s.t_eig;
  out->h2d_bytes = s.h2d;
  out->d2h_bytes = s.d2h;
}

// ============================================================ distributed
// Scene-sharded EM.  A group is the ranks one process
// drives: one rank per GPU over NCCL (ctx->comm_obj = NcclComm, the caller
// passes the full model x and its scene shard y), or G virtual ranks on one
// device (fcpd_create_loopback: LoopComm; the caller passes the full scene,
// split here into G contiguous shards).  Every rank keeps the whole model
// for the E-step, owns M_r = ⌈M/G⌉ model rows for the M-step, and its
// scene shard.  Per iteration, in the common case, three collectives:
//   reduce-scatter of the pass-2 row sums (5 doubles per row),
//   all-reduce of z (3K doubles + the flagged-row count),
//   all-gather of x̃ (float4 per row; the σ² partials ride in .w),
// plus, only when some row's global mass is too small for the fp32 fast
// path, the exact fallback exchange under a conditional graph node.

std::vector<fcpd_ctx*> group_ranks(fcpd_ctx* lead) {
  std::vector<fcpd_ctx*> r{lead};
  for (fcpd_ctx* c : lead->loop_ranks) r.push_back(c);
  return r;
}

// per-rank own-row views of the distributed E-step outputs
DistRowOut dist_out(Session& s) {
  return DistRowOut{s.ptilde_y.p, s.var.p, s.log2p1.p, s.degenerate.p, s.resid4.p, s.x0.p};
}

template <typename T, typename F>
std::vector<T> per_rank(const std::vector<fcpd_ctx*>& R, F f) {
  std::vector<T> v;
  for (fcpd_ctx* c : R) v.push_back(f(c->sess));
  return v;
}

// The exact fallback for rows of tiny global mass: the flagged rows' max L
// over all columns (all-reduce MAX), the shifted fp64 sums over each rank's
// columns (reduce-scatter), their finalisation, and their z contribution.
void enqueue_fallback(const std::vector<fcpd_ctx*>& R, Comm& comm, cudaStream_t str) {
  const int64_t k = R[0]->basis.k;
  comm.all_gather(per_rank<const uint32_t*>(R, [](Session& s) {
                    return reinterpret_cast<const uint32_t*>(s.mask_own.p); }),
                  per_rank<uint32_t*>(R, [](Session& s) {
                    return reinterpret_cast<uint32_t*>(s.mask_all.p); }),
                  static_cast<size_t>(R[0]->sess.mr), str);
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    launch_fallback_max(s.mask_all.p, s.m_pad, s.xt4.p, s.y4b.p, s.n, s.fmax_all.p, s.st.p, str);
  }
  comm.all_reduce_max(per_rank<float*>(R, [](Session& s) { return s.fmax_all.p; }),
                      static_cast<size_t>(R[0]->sess.m_pad), str);
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    launch_fallback_sum(s.mask_all.p, s.m_pad, s.fmax_all.p, s.xt4.p, s.y4b.p, s.n, s.fsum_all.p,
                        s.st.p, str);
  }
  comm.reduce_scatter_sum(per_rank<const double*>(R, [](Session& s) { return s.fsum_all.p; }),
                          per_rank<double*>(R, [](Session& s) { return s.fsum_own.p; }),
                          static_cast<size_t>(5 * R[0]->sess.mr), str);
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    launch_fallback_finalize_own(s.fsum_own.p, s.fmax_all.p + s.m0, s.mask_own.p, s.mr, s.xt64.p,
                                 dist_out(s), s.ystats, s.st.p, str);
    launch_zcorr(s.qt_own.p, s.mr4, k, s.mask_own.p, s.resid4.p, s.mr, s.zcorr.p, s.st.p, str);
  }
  comm.all_reduce_sum(per_rank<double*>(R, [](Session& s) { return s.zcorr.p; }),
                      static_cast<size_t>(3 * k), str);
  for (fcpd_ctx* c : R) launch_zadd(c->sess.zfull.p, c->sess.zcorr.p, 3 * k, c->sess.st.p, str);
}

// Enqueue `body` under a device-side predicate (a conditional IF node in the
// graph being captured on `str`).  Throws if capture into the body fails;
// the caller then re-captures with the body unconditional.
void enqueue_if(cudaStream_t str, const std::function<void(cudaGraphConditionalHandle)>& set_pred,
                const std::function<void(cudaStream_t)>& body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph = nullptr;
  FCPD_CUDA(cudaStreamGetCaptureInfo(str, &cs, nullptr, &graph, nullptr, nullptr));
  if (cs != cudaStreamCaptureStatusActive) throw Failure(FCPD_ERR_CUDA, "enqueue_if: not capturing");
  cudaGraphConditionalHandle h;
  FCPD_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
  set_pred(h);
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  FCPD_CUDA(cudaStreamGetCaptureInfo(str, &cs, nullptr, &graph, &deps, &ndeps));
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  FCPD_CUDA(cudaGraphAddNode(&node, graph, deps, ndeps, &p));
  cudaGraph_t body_graph = p.conditional.phGraph_out[0];
  cudaStream_t bs = nullptr;
  FCPD_CUDA(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
  try {
    FCPD_CUDA(cudaStreamBeginCaptureToGraph(bs, body_graph, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeRelaxed));
    body(bs);
    cudaGraph_t out = nullptr;
    FCPD_CUDA(cudaStreamEndCapture(bs, &out));
  } catch (...) {
    cudaGraph_t out = nullptr;
    cudaStreamEndCapture(bs, &out);
    cudaStreamDestroy(bs);
    throw;
  }
  cudaStreamDestroy(bs);
  FCPD_CUDA(cudaStreamUpdateCaptureDependencies(str, &node, 1, cudaStreamSetCaptureDependencies));
}

void enqueue_iteration_group(fcpd_ctx* lead, cudaStream_t str, bool conditional) {
  const std::vector<fcpd_ctx*> R = group_ranks(lead);
  Comm& comm = *lead->comm_obj;
  Session& s0 = lead->sess;
  const int64_t k = lead->basis.k;
  // E-step: pass 1 is column-local; pass 2 leaves per-row sums of the local
  // columns (AoS [M_pad][5])
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    const EStepBuffers eb = estep_buffers(s, nullptr, false, s.rowsum_all.p);
    launch_estep_pass1(s.ep, eb, s.m, s.n, s.st.p, str);
    launch_estep_pass2(s.ep, eb, s.m, s.n, s.st.p, str);
  }
  comm.reduce_scatter_sum(per_rank<const double*>(R, [](Session& s) { return s.rowsum_all.p; }),
                          per_rank<double*>(R, [](Session& s) { return s.rowsum_own.p; }),
                          static_cast<size_t>(5 * s0.mr), str);
  // own rows: finalise (flagged rows queued, zero residual), z partial over
  // the own columns of Qᵀ, the local flagged count in z[3K]
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    Basis& b = c->basis;
    IterState* st = s.st.p;
    launch_row_finalize_own(s.rowsum_own.p, s.mr, s.m_valid_own, s.n_global, s.xt64.p,
                            dist_out(s), s.ystats, s.mask_own.p, st, str);
    if (s.zp.trunc)
      launch_spectral_rank(b.lam, b.lam + b.k, b.k, s.cfg.lambda_reg, s.tau, st, str);
    if (s.rowdot) {
      launch_rowdot(s.zr, s.qt_own.p, s.resid4.p, s.zpart.p, st, s.stamps.p, 1, str);
      launch_rowdot_reduce(s.zr, s.zpart.p, b.k, nullptr, nullptr, 0.0, nullptr, nullptr,
                           s.zfull.p, st, str);
    } else {
      launch_colsum(s.zp, b.q + s.m0 * b.kpad, b.kpad, s.resid4.p, s.zpart.p, st, s.stamps.p, 1,
                    str);
      launch_zsum(s.zp, s.zpart.p, s.zfull.p, st, str);
    }
    launch_put_flag_count(s.zfull.p, b.k, st, str);
  }
  comm.all_reduce_sum(per_rank<double*>(R, [](Session& s) { return s.zfull.p; }),
                      static_cast<size_t>(3 * k + 1), str);
  if (conditional) {
    enqueue_if(
        str,
        [&](cudaGraphConditionalHandle h) {
          launch_set_fallback_cond(h, s0.zfull.p, k, s0.st.p, str);
        },
        [&](cudaStream_t bs) { enqueue_fallback(R, comm, bs); });
  } else {
    enqueue_fallback(R, comm, str);
  }
  // filter, V over the own rows, transform, σ² partial packed into x̃'s .w
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    Basis& b = c->basis;
    IterState* st = s.st.p;
    launch_zfilter(s.zfull.p, b.k, b.lam, b.lam + b.k, s.cfg.lambda_reg, s.coef.p, s.g4.p, st, str);
    launch_colsum(s.vp, s.qt_own.p, s.mr4, s.g4.p, s.vpart.p, st, nullptr, 0, str);
    const int nb = launch_transform_rows(s.vp, s.vpart.p, s.m_valid_own, s.x0.p, s.xt64.p,
                                         s.xt_prev.p, s.xt4.p + s.m0, s.ptilde_y.p, s.var.p,
                                         s.sig_part.p, st, s.stamps.p, str);
    launch_sigma_local_sum(s.sig_part.p, nb, nullptr, s.xt4.p + s.m0, st, str);
  }
  comm.all_gather(per_rank<const uint32_t*>(R, [](Session& s) {
                    return reinterpret_cast<const uint32_t*>(s.xt4.p + s.m0); }),
                  per_rank<uint32_t*>(R, [](Session& s) {
                    return reinterpret_cast<uint32_t*>(s.xt4.p); }),
                  static_cast<size_t>(4 * s0.mr), str);
  for (fcpd_ctx* c : R) {
    Session& s = c->sess;
    launch_sigma_final_gathered(s.xt4.p, s.mr, comm.world, s.m, s.d, s.cfg.early_stop,
                                s.trace.p, s.st.p, s.stamps.p, str);
  }
}

// One rank's session state for its scene shard (normalised, SoA 3×n);
// xs/y statistics are the group's.
void prepare_rank(fcpd_ctx* c, int rank, int world, const std::vector<double>& xs_in, int64_t m,
                  std::vector<double> ys, int64_t n, int64_t n_global, const YStats& ystats,
                  int d, const fcpd_config& cfg, double sigma2_initial) {
  Session& s = c->sess;
  cudaStream_t str = c->stream;
  s.ready = false;
  s.dist = true;
  s.h2d = s.d2h = 0;
  s.m = m;
  s.n = n;
  s.d = d;
  s.cfg = cfg;
  s.n_global = n_global;
  s.ystats = ystats;
  s.sigma2_initial = sigma2_initial;
  if (m < world) throw Failure(FCPD_ERR_PARAMETER, "register: fewer model points than ranks");
  // internal spatial order: the full model (identical on all ranks) and the
  // local scene shard; row shards are spatial slabs
  std::vector<double> xs = xs_in;
  s.perm_x = spatial_sort_cached(xs, m, c->sort_x);
  s.perm_y = spatial_sort_cached(ys, n, c->sort_y);
  // spectral basis (each rank keeps its row shard of it)
  s.x0.ensure(3 * m);
  FCPD_CUDA(cudaMemcpyAsync(s.x0.p, xs.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice, str));
  ensure_basis(c, s, xs);
  c->basis.perm = s.perm_x;
  Basis& b = c->basis;
  // shard geometry
  s.mr = (m + world - 1) / world;
  s.m_pad = s.mr * world;
  s.m0 = s.mr * rank;
  s.m_valid_own = std::max<int64_t>(0, std::min<int64_t>(s.mr, m - s.m0));
  if (s.m_valid_own < 1) throw Failure(FCPD_ERR_PARAMETER, "register: empty model shard");
  if (s.mr < 2) throw Failure(FCPD_ERR_PARAMETER, "register: fewer than 2 model rows per rank");
  s.mr4 = (s.mr + 3) / 4 * 4;
  const int64_t mr = s.mr;
  std::vector<double> own(3 * mr, 0.0);
  for (int cc = 0; cc < 3; ++cc)
    for (int64_t i = 0; i < s.m_valid_own; ++i) own[cc * mr + i] = xs[cc * m + s.m0 + i];
  s.release_graph();
  s.x0.ensure(3 * mr);
  s.xt64.ensure(3 * mr);
  s.xt_prev.ensure(3 * mr);
  s.ptilde_y.ensure(3 * mr);
  s.var.ensure(mr);
  s.log2p1.ensure(mr);
  s.degenerate.ensure(mr);
  s.resid4.ensure(mr);
  FCPD_CUDA(cudaMemcpyAsync(s.x0.p, own.data(), sizeof(double) * 3 * mr, cudaMemcpyHostToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.xt64.p, s.x0.p, sizeof(double) * 3 * mr, cudaMemcpyDeviceToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.xt_prev.p, s.x0.p, sizeof(double) * 3 * mr, cudaMemcpyDeviceToDevice, str));
  FCPD_CUDA(cudaMemsetAsync(s.resid4.p, 0, sizeof(float4) * mr, str));
  // full model (float4, padded far away) and the local scene
  std::vector<float4> x4(s.m_pad, make_float4(3.0e18f, 3.0e18f, 3.0e18f, 0.f)), y4(n);
  for (int64_t i = 0; i < m; ++i)
    x4[i] = make_float4(static_cast<float>(xs[i]), static_cast<float>(xs[m + i]),
                        static_cast<float>(xs[2 * m + i]), 0.f);
  for (int64_t i = 0; i < n; ++i)
    y4[i] = make_float4(static_cast<float>(ys[i]), static_cast<float>(ys[n + i]),
                        static_cast<float>(ys[2 * n + i]), 0.f);
  s.xt4.ensure(s.m_pad);
  s.y4b.ensure(n);
  FCPD_CUDA(cudaMemcpyAsync(s.xt4.p, x4.data(), sizeof(float4) * s.m_pad, cudaMemcpyHostToDevice, str));
  FCPD_CUDA(cudaMemcpyAsync(s.y4b.p, y4.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, str));
  s.h2d += (sizeof(double) * 3 + sizeof(float4)) * (m + n);
  // E-step scratch over all M rows / local columns
  s.ep = make_estep_plan(m, n, c->sm_count);
  s.b2.ensure(n);
  s.pt1.ensure(n);
  s.col_flags.ensure(n);
  s.row_flags.ensure(m);
  s.rowsum_all.ensure(5 * s.m_pad);
  // rows in [M, M_pad) are never written: zero once
  FCPD_CUDA(cudaMemsetAsync(s.rowsum_all.p, 0, sizeof(double) * 5 * s.m_pad, str));
  s.rowsum_own.ensure(5 * mr);
  s.fsum_all.ensure(5 * s.m_pad);
  s.fsum_own.ensure(5 * mr);
  s.mask_own.ensure(mr);
  s.mask_all.ensure(s.m_pad);
  s.fmax_all.ensure(s.m_pad);
  FCPD_CUDA(cudaMemsetAsync(s.mask_own.p, 0, sizeof(int32_t) * mr, str));
  alloc_estep(s, m, n, str);
  // basis shard: Q rows [m0, m0+m_valid) in place; Qᵀ columns copied compact
  s.qt_own.ensure(static_cast<size_t>(b.k) * s.mr4);
  FCPD_CUDA(cudaMemsetAsync(s.qt_own.p, 0, sizeof(float) * b.k * s.mr4, str));
  const int64_t cols = std::min<int64_t>(mr, b.mpad - s.m0);
  if (cols > 0)
    FCPD_CUDA(cudaMemcpy2DAsync(s.qt_own.p, sizeof(float) * s.mr4, b.qt + s.m0,
                                sizeof(float) * b.mpad, sizeof(float) * cols, b.k,
                                cudaMemcpyDeviceToDevice, str));
  s.zp = make_colsum_plan(s.m_valid_own, b.k, c->sm_count);
  s.vp = make_colsum_plan(b.k, mr, c->sm_count);
  // spectral truncation as on one GPU (the same cut on every rank: it
  // depends only on λ and the σ² every rank computes identically)
  s.tau = s.cfg.spectral_tau;
  if (4.0 * static_cast<double>(m) * static_cast<double>(b.k) < 64.0 * (1 << 20)) s.tau = 0.0;
  if (const char* e = std::getenv("FCPD_SPECTRAL_TAU")) s.tau = std::atof(e);
  s.zp.trunc = s.tau > 0.0 ? 1 : 0;
  s.vp.trunc = s.tau > 0.0 ? 2 : 0;
  {
    const char* zpass = std::getenv("FCPD_ZPASS");
    s.rowdot = !(zpass && std::string(zpass) == "colsum");
    s.zr = make_rowdot_plan(b.k, s.m_valid_own, s.mr4, c->sm_count);
    s.zr.g.trunc = s.zp.trunc;
  }
  s.zpart.ensure(std::max(s.zp.part_doubles(), s.rowdot ? s.zr.part_doubles() : size_t(0)));
  s.vpart.ensure(s.vp.part_doubles());
  s.zfull.ensure(3 * b.k + 1);
  s.zcorr.ensure(3 * b.k);
  s.coef.ensure(3 * b.k);
  s.g4.ensure(b.kpad);
  s.sig_part.ensure(transform_sigma_blocks(mr));
  s.sig_local.ensure(1);
  s.st.ensure(1);
  s.capacity = std::max(cfg.iterations, 1);
  s.trace.ensure(s.capacity);
  s.stamps.ensure(4 * static_cast<size_t>(s.capacity));
  reset_state(c, s, sigma2_initial);
  FCPD_CUDA(cudaMemsetAsync(s.coef.p, 0, sizeof(double) * 3 * b.k, str));
  FCPD_CUDA(cudaStreamSynchronize(str));
}

// The top-K basis of a low-rank rank group (configs 2–4 sharded): one
// randomized eigensolve for the group with its Φ·V products row-sharded
// over the ranks (topk.cu gram_matmul_sharded: each rank its M/G rows, an
// all-gather), installed in every rank's context under the key
// ensure_basis looks up, so prepare_rank finds it cached.  Returns the
// solve's wall time (0: not this path, or already cached).
double group_topk_basis(fcpd_ctx* lead, const std::vector<fcpd_ctx*>& R,
                        const std::vector<double>& xs_in, int64_t m, int d,
                        const fcpd_config& cfg) {
  Comm& comm = *lead->comm_obj;
  if (comm.world < 2 || cfg.variant != FCPD_VARIANT_FAST_LOWRANK) return 0.0;
  int64_t topk_min = kDenseEigLimitLowrank;
  if (const char* e = std::getenv("FCPD_TOPK_MIN_M")) topk_min = std::atoll(e);
  if (m <= topk_min) return 0.0;
  if (!(cfg.beta > 0.0)) throw Failure(FCPD_ERR_PARAMETER, "build_gram: beta must be positive");
  const int64_t rank = lowrank_rank(cfg.rank_fraction, m);
  std::vector<double> xs = xs_in;
  spatial_sort_cached(xs, m, lead->sort_x);  // the order prepare_rank uses
  uint64_t h = fnv1a(xs.data(), sizeof(double) * xs.size());
  h = fnv1a(&m, sizeof m, h);
  h = fnv1a(&rank, sizeof rank, h);
  std::vector<std::vector<double>> need(R.size(), std::vector<double>(1, 0.0));
  for (size_t i = 0; i < R.size(); ++i) {
    const Basis& b = R[i]->basis;
    const bool hit = b.q && b.key_hash == h && b.key_beta == cfg.beta && b.m == m &&
                     b.k == rank && b.key_variant == cfg.variant;
    need[i][0] = hit ? 0.0 : 1.0;
  }
  comm.host_all_reduce(need, true, lead->stream);  // every rank takes the same branch
  if (need[0][0] == 0.0) return 0.0;
  const auto t1 = Clock::now();
  DevBuf<double> xd;
  xd.ensure(3 * static_cast<size_t>(m));
  FCPD_CUDA(cudaMemcpyAsync(xd.p, xs.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice,
                            lead->stream));
  GramShards sh;
  sh.comm = &comm;
  std::vector<Basis*> also;
  for (size_t i = 0; i < R.size(); ++i) {
    sh.ranks.push_back(lead->loop_ranks.empty() ? lead->rank : static_cast<int>(i));
    R[i]->basis.release();
    if (i > 0) also.push_back(&R[i]->basis);
  }
  topk_eigensolve(lead->solver, lead->blas, xd.p, m, d, cfg.beta, rank, topk_iterations(),
                  topk_adaptive(), cfg.seed, lead->basis, lead->stream, nullptr, nullptr, &sh,
                  &also);
  FCPD_CUDA(cudaStreamSynchronize(lead->stream));
  xd.release();
  const double t = since(t1);
  for (fcpd_ctx* c : R) {
    Basis& b = c->basis;
    upload_lambda(b, false, lead->stream);
    b.key_hash = h;
    b.key_beta = cfg.beta;
    b.key_variant = cfg.variant;
    b.t_gram = 0.0;
    b.t_eig = t;
  }
  FCPD_CUDA(cudaStreamSynchronize(lead->stream));
  return t;
}

// shards: per local rank, (pointer to its SoA scene shard, count)
void session_begin_group(fcpd_ctx* lead, const double* x, int64_t m,
                         const std::vector<std::pair<const double*, int64_t>>& shards, int d,
                         const fcpd_config& cfg) {
  const std::vector<fcpd_ctx*> R = group_ranks(lead);
  Comm& comm = *lead->comm_obj;
  const int G = comm.world;
  const auto t0 = Clock::now();
  for (size_t i = 0; i < R.size(); ++i)
    validate_register(x, m, shards[i].first, shards[i].second, d, cfg);
  // global scene size and normalize_pair statistics (pointset.hpp:124-148)
  std::vector<std::vector<double>> red(R.size(), std::vector<double>(4, 0.0));
  for (size_t i = 0; i < R.size(); ++i) {
    const double* y = shards[i].first;
    const int64_t n = shards[i].second;
    red[i][0] = static_cast<double>(n);
    for (int c = 0; c < d; ++c)
      for (int64_t j = 0; j < n; ++j) red[i][1 + c] += y[c * n + j];
  }
  comm.host_all_reduce(red, false, lead->stream);
  const int64_t n_global = static_cast<int64_t>(red[0][0]);
  double center[3] = {0.0, 0.0, 0.0}, scale = 1.0;
  if (cfg.normalize) {
    const double total = static_cast<double>(m + n_global);
    for (int c = 0; c < d; ++c) {
      double sx = 0.0;
      for (int64_t j = 0; j < m; ++j) sx += x[c * m + j];
      center[c] = (sx + red[0][1 + c]) / total;
    }
    std::vector<std::vector<double>> sc(R.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < R.size(); ++i) {
      const double* y = shards[i].first;
      const int64_t n = shards[i].second;
      double v = 0.0;
      for (int c = 0; c < d; ++c) {
        for (int64_t j = 0; j < m; ++j) v = std::max(v, std::fabs(x[c * m + j] - center[c]));
        for (int64_t j = 0; j < n; ++j) v = std::max(v, std::fabs(y[c * n + j] - center[c]));
      }
      sc[i][0] = v;
    }
    comm.host_all_reduce(sc, true, lead->stream);
    scale = sc[0][0] > 0.0 ? sc[0][0] : 1.0;
  }
  auto norm = [&](const double* p, int64_t cnt) {
    std::vector<double> o(3 * cnt, 0.0);
    for (int c = 0; c < d; ++c)
      for (int64_t j = 0; j < cnt; ++j)
        o[c * cnt + j] = cfg.normalize ? (p[c * cnt + j] - center[c]) / scale : p[c * cnt + j];
    return o;
  };
  const std::vector<double> xs = norm(x, m);
  std::vector<std::vector<double>> ys(R.size());
  std::vector<std::vector<double>> yst(R.size(), std::vector<double>(4, 0.0));
  for (size_t i = 0; i < R.size(); ++i) {
    ys[i] = norm(shards[i].first, shards[i].second);
    const int64_t n = shards[i].second;
    for (int c = 0; c < 3; ++c)
      for (int64_t j = 0; j < n; ++j) yst[i][c] += ys[i][c * n + j];
    for (int64_t j = 0; j < n; ++j)
      yst[i][3] += ys[i][j] * ys[i][j] + ys[i][n + j] * ys[i][n + j] +
                   ys[i][2 * n + j] * ys[i][2 * n + j];
  }
  comm.host_all_reduce(yst, false, lead->stream);
  const double ng = static_cast<double>(n_global);
  YStats ystats{};
  for (int c = 0; c < 3; ++c) ystats.mean[c] = yst[0][c] / ng;
  ystats.sq_mean = yst[0][3] / ng;
  // init_sigma2 (registration.hpp:59-69) from the global statistics
  double sigma2_initial = 0.0;
  {
    double fx = 0.0, dot = 0.0;
    for (int c = 0; c < d; ++c) {
      double sx = 0.0;
      for (int64_t j = 0; j < m; ++j) {
        fx += xs[c * m + j] * xs[c * m + j];
        sx += xs[c * m + j];
      }
      dot += sx * yst[0][c];
    }
    const double md = static_cast<double>(m);
    sigma2_initial = std::max((md * yst[0][3] + ng * fx - 2.0 * dot) / (static_cast<double>(d) * md * ng), 0.0);
  }
  if (cfg.iterations > 0 && !(cfg.omega >= 0.0 && cfg.omega < 1.0))
    throw Failure(FCPD_ERR_NUMERIC, "register: iteration 0: posterior: omega must lie in [0, 1)");
  const double t_group_eig = group_topk_basis(lead, R, xs, m, d, cfg);
  for (size_t i = 0; i < R.size(); ++i) {
    const int rank = lead->loop_ranks.empty() ? lead->rank : static_cast<int>(i);
    prepare_rank(R[i], rank, G, xs, m, ys[i], shards[i].second, n_global, ystats, d, cfg,
                 sigma2_initial);
    Session& s = R[i]->sess;
    for (int c = 0; c < 3; ++c) s.center[c] = center[c];
    s.scale = scale;
    if (t_group_eig > 0.0) {  // built above for the group, not reused from a cache
      s.basis_reused = false;
      s.t_eig = t_group_eig;
    }
  }
  // one EM iteration of the whole group as a CUDA graph on the lead stream;
  // the fallback exchange behind a conditional node where the backend
  // allows it (else, or if capturing into the node fails, unconditional)
  cudaStream_t str = lead->stream;
  bool conditional = comm.conditional_ok();
  if (const char* e = std::getenv("FCPD_DIST_CONDITIONAL")) conditional = std::atoi(e) != 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    cudaGraph_t g = nullptr;
    FCPD_CUDA(cudaStreamBeginCapture(str, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_iteration_group(lead, str, conditional);
    } catch (const Failure&) {
      cudaStreamEndCapture(str, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      if (!conditional) throw;
      conditional = false;  // retry with the fallback exchange unconditional
      continue;
    }
    FCPD_CUDA(cudaStreamEndCapture(str, &g));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      cudaGetLastError();
      if (!conditional) FCPD_CUDA(ie);
      conditional = false;
      continue;
    }
    lead->sess.graph = exec;
    break;
  }
  lead->sess.dist_conditional = conditional;
  lead->sess.t_setup_host = since(t0);
  lead->sess.launched = 0;
  lead->sess.ready = true;
}

void session_begin_dist(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n,
                        int d, const fcpd_config& cfg) {
  std::vector<std::pair<const double*, int64_t>> shards;
  std::vector<std::vector<double>> store;
  if (ctx->loop_ranks.empty()) {
    shards.push_back({y, n});  // NCCL: this rank's scene shard
  } else {
    // loopback group: the full scene, split into contiguous shards as the
    // NCCL callers do (bench.py: rows [r·N/G, (r+1)·N/G))
    const int G = ctx->comm_obj->world;
    if (n < G) throw Failure(FCPD_ERR_PARAMETER, "register: fewer scene points than ranks");
    for (int r = 0; r < G; ++r) {
      const int64_t a = r * n / G, b = (r + 1) * n / G;
      std::vector<double> sh(static_cast<size_t>(d) * (b - a));
      for (int c = 0; c < d; ++c)
        std::memcpy(&sh[c * (b - a)], y + c * n + a, sizeof(double) * (b - a));
      store.push_back(std::move(sh));
    }
    for (int r = 0; r < G; ++r)
      shards.push_back({store[r].data(), (r + 1) * n / G - r * n / G});
  }
  session_begin_group(ctx, x, m, shards, d, cfg);
}

// gather the own-row SoA blocks (stride mr) of every rank into a full SoA
// M×d on the host (every rank of the group takes part)
void gather_rows(fcpd_ctx* lead, const std::function<const double*(Session&)>& own,
                 double* out_full, int d) {
  const std::vector<fcpd_ctx*> R = group_ranks(lead);
  Comm& comm = *lead->comm_obj;
  const int G = comm.world;
  Session& s0 = lead->sess;
  for (fcpd_ctx* c : R) c->sess.stage.ensure(static_cast<size_t>(3) * c->sess.mr * G);
  comm.all_gather(per_rank<const uint32_t*>(R, [&](Session& s) {
                    return reinterpret_cast<const uint32_t*>(own(s)); }),
                  per_rank<uint32_t*>(R, [](Session& s) {
                    return reinterpret_cast<uint32_t*>(s.stage.p); }),
                  static_cast<size_t>(3 * s0.mr * 2), lead->stream);
  std::vector<double> h(static_cast<size_t>(3) * s0.mr * G);
  FCPD_CUDA(cudaMemcpyAsync(h.data(), s0.stage.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                            lead->stream));
  FCPD_CUDA(cudaStreamSynchronize(lead->stream));
  s0.d2h += sizeof(double) * 3 * s0.mr;
  for (int r = 0; r < G; ++r)
    for (int c = 0; c < d; ++c)
      for (int64_t i = 0; i < s0.mr; ++i) {
        const int64_t row = r * s0.mr + i;
        if (row < s0.m) out_full[c * s0.m + row] = h[(static_cast<size_t>(r) * 3 + c) * s0.mr + i];
      }
}

void session_read_dist(fcpd_ctx* ctx, fcpd_result* out, double wall) {
  const std::vector<fcpd_ctx*> R = group_ranks(ctx);
  Comm& comm = *ctx->comm_obj;
  Session& s = ctx->sess;
  cudaStream_t str = ctx->stream;
  std::vector<IterState> hs(R.size());
  for (size_t i = 0; i < R.size(); ++i)
    FCPD_CUDA(cudaMemcpyAsync(&hs[i], R[i]->sess.st.p, sizeof(IterState), cudaMemcpyDeviceToHost,
                              str));
  FCPD_CUDA(cudaStreamSynchronize(str));
  const IterState& h = hs[0];
  if (h.err_code != 0) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", h.err_value);
    const std::string what = h.err_code == kDevSolveDiag
                                 ? "solve_fast: lambda_i + lambda*sigma2 not positive"
                                 : std::string("update_sigma2: negative variance ") + buf;
    throw Failure(FCPD_ERR_NUMERIC, "register: iteration " + std::to_string(h.err_iter) + ": " + what);
  }
  std::vector<std::vector<double>> deg(R.size(), std::vector<double>(1, 0.0));
  for (size_t i = 0; i < R.size(); ++i) deg[i][0] = static_cast<double>(hs[i].degenerate_rows);
  comm.host_all_reduce(deg, false, str);  // own-row counts → global
  if (!out) return;
  if (out->correspondence)
    throw Failure(FCPD_ERR_PARAMETER, "register: correspondence output is single-GPU only");
  const int run = h.iters_run;
  const int d = s.d;
  Basis& b = ctx->basis;
  out->iterations_run = run;
  out->basis_reused = s.basis_reused ? 1 : 0;
  out->sigma2_initial = s.sigma2_initial;
  out->degenerate_rows = static_cast<int64_t>(deg[0][0]);
  out->spectral_rank = s.zp.trunc && h.keff > 0 ? std::min<int64_t>(h.keff, b.k) : b.k;
  out->sigma2_clamps = h.sigma2_clamps;
  if (out->sigma2_trace && run > 0)
    FCPD_CUDA(cudaMemcpyAsync(out->sigma2_trace, s.trace.p, sizeof(double) * run,
                              cudaMemcpyDeviceToHost, str));
  std::vector<double> xt(3 * s.m, 0.0);
  gather_rows(ctx, [](Session& q) { return static_cast<const double*>(q.xt64.p); }, xt.data(), 3);
  const std::vector<int64_t>& px = s.perm_x;  // sorted row k ↔ original row px[k]
  if (out->transformed)
    for (int c = 0; c < d; ++c)
      for (int64_t k = 0; k < s.m; ++k)
        out->transformed[c * s.m + px[k]] =
            s.cfg.normalize ? xt[c * s.m + k] * s.scale + s.center[c] : xt[c * s.m + k];
  if (out->coefficients) {
    if (s.zp.trunc && run > 0) {  // the iterations streamed a truncated basis
      for (fcpd_ctx* c : R) {
        Session& q = c->sess;
        Basis& qb = c->basis;
        launch_colsum(q.zp, qb.q + q.m0 * qb.kpad, qb.kpad, q.resid4.p, q.zpart.p, nullptr,
                      nullptr, 0, str);
        launch_zsum(q.zp, q.zpart.p, q.zfull.p, nullptr, str);
      }
      comm.all_reduce_sum(per_rank<double*>(R, [](Session& q) { return q.zfull.p; }),
                          static_cast<size_t>(3 * b.k), str);
      for (fcpd_ctx* c : R)
        launch_zcoef_full(c->sess.zfull.p, c->basis.k, c->basis.lam, c->sess.cfg.lambda_reg,
                          c->sess.coef.p, c->sess.st.p, str);
    }
    for (fcpd_ctx* c : R) {
      Session& q = c->sess;
      pack_coef_kernel<<<ceil_div(c->basis.k, 256), 256, 0, str>>>(q.coef.p, c->basis.k, q.g4.p);
      FCPD_LAUNCH_CHECK();
      launch_colsum(q.vp, q.qt_own.p, q.mr4, q.g4.p, q.vpart.p, nullptr, nullptr, 0, str);
      launch_vreduce_add(q.vp, q.vpart.p, nullptr, 3, q.ptilde_y.p, str);
    }
    std::vector<double> w(3 * s.m, 0.0);
    gather_rows(ctx, [](Session& q) { return static_cast<const double*>(q.ptilde_y.p); },
                w.data(), 3);
    for (int c = 0; c < d; ++c)
      for (int64_t k = 0; k < s.m; ++k) out->coefficients[c * s.m + px[k]] = w[c * s.m + k];
  }
  std::vector<uint64_t> stamps(4 * static_cast<size_t>(std::max(run, 1)));
  if (run > 0)
    FCPD_CUDA(cudaMemcpyAsync(stamps.data(), s.stamps.p, sizeof(uint64_t) * 4 * run,
                              cudaMemcpyDeviceToHost, str));
  FCPD_CUDA(cudaStreamSynchronize(str));
  double tc = 0.0, ti = 0.0;
  for (int it = 0; it < run; ++it) {
    tc += 1e-9 * static_cast<double>(stamps[4 * it + 1] - stamps[4 * it]);
    ti += 1e-9 * static_cast<double>(stamps[4 * it + 2] - stamps[4 * it + 1]);
  }
  fcpd_timing& t = out->timing;
  t.t_c = tc;
  t.t_eig = s.t_eig;
  t.t_iter = ti;
  t.t_f = t.t_eig + t.t_iter;
  t.t_o = std::max(wall - t.t_c - t.t_f, 0.0);
  t.t_total = t.t_c + t.t_f + t.t_o;
  t.t_setup = s.t_gram + s.t_eig;
  out->h2d_bytes = s.h2d;
  out->d2h_bytes = s.d2h;
}

}  // namespace

CtxHandles ctx_handles(fcpd_ctx* ctx) {
  return CtxHandles{ctx->device, ctx->stream, ctx->blas, ctx->solver};
}

int ctx_guarded(fcpd_ctx* ctx, const std::function<void()>& f) { return guarded(ctx, f); }

}  // namespace fcpd

// ============================================================== C ABI

using namespace fcpd;

extern "C" {

void fcpd_config_default(fcpd_config* cfg) {
  if (!cfg) return;
  cfg->omega = 0.7;
  cfg->beta = 2.0;
  cfg->lambda_reg = 10.0;
  cfg->iterations = 100;
  cfg->variant = FCPD_VARIANT_FAST;
  cfg->rank_fraction = 0.1;
  cfg->seed = 0;
  cfg->normalize = 1;
  cfg->early_stop = 0;
  cfg->pad0 = 0;
  cfg->spectral_tau = 1e-10;
}

const char* fcpd_version(void) { return "fcpd-b200 0.1 (sm_100a)"; }

int fcpd_create(fcpd_ctx** out, int device) {
  if (!out) return FCPD_ERR_PARAMETER;
  *out = nullptr;
  auto* ctx = new (std::nothrow) fcpd_ctx();
  if (!ctx) return FCPD_ERR_OOM;
  ctx->device = device;
  try {
    FCPD_CUDA(cudaSetDevice(device));
    int sms = 0;
    FCPD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    ctx->sm_count = sms;
    FCPD_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    if (cusolverDnCreate(&ctx->solver) != CUSOLVER_STATUS_SUCCESS)
      throw Failure(FCPD_ERR_CUDA, "cusolverDnCreate failed");
    if (cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS)
      throw Failure(FCPD_ERR_CUDA, "cublasCreate failed");
  } catch (const Failure& e) {
    static thread_local std::string last;
    last = e.what();
    delete ctx;
    return e.code;
  }
  *out = ctx;
  return FCPD_OK;
}

int fcpd_nccl_unique_id(uint8_t* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!out128) return FCPD_ERR_PARAMETER;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FCPD_ERR_NCCL;
  std::memcpy(out128, &id, sizeof id);
  return FCPD_OK;
}

int fcpd_create_dist(fcpd_ctx** out, int device, int rank, int world, const uint8_t* id128) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world) return FCPD_ERR_PARAMETER;
  int rc = fcpd_create(out, device);
  if (rc) return rc;
  fcpd_ctx* ctx = *out;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) {
    fcpd_destroy(ctx);
    *out = nullptr;
    return FCPD_ERR_NCCL;
  }
  ctx->rank = rank;
  ctx->world = world;
  ctx->comm_obj = std::make_unique<NcclComm>(ctx->comm, world);
  return FCPD_OK;
}

int fcpd_create_loopback(fcpd_ctx** out, int device, int world) {
  if (!out || world < 1 || world > kMaxLoopRanks) return FCPD_ERR_PARAMETER;
  int rc = fcpd_create(out, device);
  if (rc) return rc;
  fcpd_ctx* lead = *out;
  for (int r = 1; r < world; ++r) {
    fcpd_ctx* c = nullptr;
    rc = fcpd_create(&c, device);
    if (rc) {
      fcpd_destroy(lead);
      *out = nullptr;
      return rc;
    }
    c->rank = r;
    c->world = world;
    lead->loop_ranks.push_back(c);
  }
  lead->rank = 0;
  lead->world = world;
  lead->comm_obj = std::make_unique<LoopComm>(world);
  return FCPD_OK;
}

int fcpd_world(const fcpd_ctx* ctx, int32_t* rank, int32_t* world) {
  if (!ctx) return FCPD_ERR_PARAMETER;
  if (rank) *rank = ctx->rank;
  if (world) *world = ctx->world;
  return FCPD_OK;
}

void fcpd_destroy(fcpd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  ctx->sess.release();
  ctx->basis.release();
  for (fcpd_ctx* c : ctx->loop_ranks) fcpd_destroy(c);
  ctx->loop_ranks.clear();
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  if (ctx->blas) cublasDestroy(ctx->blas);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* fcpd_last_error(const fcpd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* fcpd_stream(fcpd_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int32_t fcpd_kernels_per_iteration(const fcpd_ctx* ctx) {
  // single GPU: prologue, col, col-combine, col-fallback, row, row-combine,
  // row-fallback, Qᵀ·R, z-reduce/filter, Q·g, transform/σ²-rows, σ²-final.
  // distributed: prologue, col, col-combine, col-fallback, row, row-sum,
  // finalize-own, fb-max, fb-sum, fb-finalize, Qᵀ·R, z-sum, z-filter, Q·g,
  // transform, σ²-local, σ²-final (+ 7 NCCL collectives).
  // Tile culling adds 4: model-tile boxes, pass-1 list, scene-tile b range,
  // pass-2 list.
  if (!ctx) return 0;
  const Session& s = ctx->sess;
  const bool culling = s.cull && s.xlo.p && s.ylo.p && s.wl1_tiles.p;
  const int e = estep_kernels(culling, s.dist);
  if (s.dist) {
    // per rank: finalize-own, (spectral rank,) z pass + reduce, flag count,
    // z filter, Q·g, transform, σ² partial, σ² final; the fallback exchange's
    // fb-max, fb-sum, fb-finalize, z correction, z add only when it is not
    // behind the conditional node (then its predicate kernel instead); a
    // loopback group adds its three collective kernels
    const int ranks = 1 + static_cast<int>(ctx->loop_ranks.size());
    return ranks * (e + 9 + (s.zp.trunc ? 1 : 0) + (s.dist_conditional ? 0 : 5)) +
           (s.dist_conditional ? 1 : 0) + (ctx->loop_ranks.empty() ? 0 : 3);
  }
  if (s.small) return 1;  // the whole iteration (small_iter_kernel)
  // fused M-step: one kernel for rank, Qᵀ·R, filter, Q·g, transform and σ²
  if (s.mfused) return e + 1;
  // streaming: (spectral rank,) Qᵀ·R, z-reduce/filter, Q·g, transform, σ²
  return e + 5 + (s.zp.trunc ? 1 : 0);
}

int fcpd_register(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n,
                  int32_t d, const fcpd_config* cfg, fcpd_result* out) {
  return guarded(ctx, [&] {
    if (!cfg) throw Failure(FCPD_ERR_PARAMETER, "register: null config");
    const auto t0 = Clock::now();
    session_begin(ctx, x, m, y, n, d, *cfg);
    session_run(ctx, cfg->iterations);
    FCPD_CUDA(cudaStreamSynchronize(ctx->stream));
    session_read(ctx, out, since(t0));
  });
}

int fcpd_session_begin(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n,
                       int32_t d, const fcpd_config* cfg) {
  return guarded(ctx, [&] {
    if (!cfg) throw Failure(FCPD_ERR_PARAMETER, "session: null config");
    session_begin(ctx, x, m, y, n, d, *cfg);
  });
}

int fcpd_session_run(fcpd_ctx* ctx, int32_t iterations) {
  return guarded(ctx, [&] { session_run(ctx, iterations); });
}

int fcpd_session_sync(fcpd_ctx* ctx) {
  return guarded(ctx, [&] { FCPD_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int fcpd_session_read(fcpd_ctx* ctx, fcpd_result* out) {
  return guarded(ctx, [&] { session_read(ctx, out, 0.0); });
}

int fcpd_session_profile(fcpd_ctx* ctx, int32_t iterations, double* ms_per_phase) {
  return guarded(ctx, [&] {
    Session& s = ctx->sess;
    if (!s.ready) throw Failure(FCPD_ERR_PARAMETER, "session: not started");
    if (s.dist) throw Failure(FCPD_ERR_PARAMETER, "session_profile: single-GPU sessions only");
    if (iterations < 1 || s.launched + iterations > s.capacity)
      throw Failure(FCPD_ERR_PARAMETER, "session: more iterations than cfg.iterations");
    cudaEvent_t ev[7];
    for (auto& e : ev) FCPD_CUDA(cudaEventCreate(&e));
    double acc[6] = {0, 0, 0, 0, 0, 0};
    // every profiled iteration starts from a cold L2 (a 256 MB write, more
    // than the 126 MB L2), so the phase times are HBM-honest
    DevBuf<uint8_t> flush;
    flush.ensure(size_t(256) << 20);
    for (int it = 0; it < iterations; ++it) {
      FCPD_CUDA(cudaMemsetAsync(flush.p, it & 0xff, size_t(256) << 20, ctx->stream));
      enqueue_iteration(ctx, s, ev);
      ++s.launched;
      FCPD_CUDA(cudaEventSynchronize(ev[6]));
      for (int p = 0; p < 6; ++p) {
        float ms = 0.f;
        FCPD_CUDA(cudaEventElapsedTime(&ms, ev[p], ev[p + 1]));
        acc[p] += ms;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    flush.release();
    for (int p = 0; p < 6; ++p) ms_per_phase[p] = acc[p] / iterations;
  });
}

int fcpd_estep(fcpd_ctx* ctx, const double* xt, int64_t m, const double* y, int64_t n,
               int32_t d, double omega, double sigma2, double* ptilde_y, double* p1, double* var,
               int32_t* degenerate, double* pt1, int32_t* clamped) {
  return guarded(ctx, [&] {
    if (m <= 0 || n <= 0) throw Failure(FCPD_ERR_PARAMETER, "posterior: empty point set");
    if (d < 1 || d > 3) throw Failure(FCPD_ERR_DIMENSION, "posterior: the B200 path supports D <= 3");
    if (!(omega >= 0.0 && omega < 1.0))
      throw Failure(FCPD_ERR_PARAMETER, "posterior: omega must lie in [0, 1)");
    Session& s = ctx->sess;
    s.ready = false;
    s.m = m;
    s.n = n;
    s.d = d;
    fcpd_config_default(&s.cfg);
    s.cfg.omega = omega;
    std::vector<double> xs(3 * m, 0.0), ys(3 * n, 0.0);
    for (int c = 0; c < d; ++c) {
      std::memcpy(&xs[c * m], xt + c * m, sizeof(double) * m);
      std::memcpy(&ys[c * n], y + c * n, sizeof(double) * n);
    }
    s.dist = false;
    s.perm_x = spatial_sort(xs, m);  // internal spatial order (tile culling)
    s.perm_y = spatial_sort(ys, n);
    prepare_buffers(ctx, s, xs, ys, 1, false);
    reset_state(ctx, s, sigma2);
    const EStepBuffers eb = estep_buffers(s, s.pt1.p, false);
    launch_estep(s.ep, eb, m, n, s.st.p, ctx->stream);
    std::vector<double> pty(3 * m), lp(m), vr(m), pc(n);
    std::vector<int32_t> dg(m);
    cudaStream_t str = ctx->stream;
    FCPD_CUDA(cudaMemcpyAsync(pty.data(), s.ptilde_y.p, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaMemcpyAsync(lp.data(), s.log2p1.p, sizeof(double) * m, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaMemcpyAsync(vr.data(), s.var.p, sizeof(double) * m, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaMemcpyAsync(dg.data(), s.degenerate.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaMemcpyAsync(pc.data(), s.pt1.p, sizeof(double) * n, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaStreamSynchronize(str));
    // undo the spatial order: sorted row k ↔ original row perm_x[k]
    const std::vector<int64_t>& px = s.perm_x;
    for (int64_t k = 0; k < m; ++k) {
      const int64_t i = px[k];
      if (ptilde_y)
        for (int c = 0; c < d; ++c) ptilde_y[c * m + i] = pty[c * m + k];
      if (p1) p1[i] = std::exp2(lp[k]);
      if (var) var[i] = vr[k];
      if (degenerate) degenerate[i] = dg[k];
    }
    if (pt1)
      for (int64_t j = 0; j < n; ++j) pt1[s.perm_y[j]] = pc[j];
    if (clamped) *clamped = sigma2 < kSigma2Floor ? 1 : 0;
  });
}

int fcpd_posterior_dense(fcpd_ctx* ctx, const double* xt, int64_t m, const double* y, int64_t n,
                         int32_t d, double omega, double sigma2, int32_t row_constrain, double* p,
                         int32_t* clamped, int64_t* degenerate_rows, int64_t* n_degenerate) {
  std::vector<int32_t> deg(m > 0 ? m : 1);
  return guarded(ctx, [&] {
    if (m <= 0 || n <= 0) throw Failure(FCPD_ERR_PARAMETER, "posterior: empty point set");
    if (d < 1 || d > 3) throw Failure(FCPD_ERR_DIMENSION, "posterior: the B200 path supports D <= 3");
    if (!(omega >= 0.0 && omega < 1.0))
      throw Failure(FCPD_ERR_PARAMETER, "posterior: omega must lie in [0, 1)");
    if (static_cast<double>(m) * static_cast<double>(n) > 4e9)
      throw Failure(FCPD_ERR_PARAMETER, "posterior: dense output limited to M*N <= 4e9");
    cudaStream_t str = ctx->stream;
    DevBuf<double> xd, yd, dp;
    DevBuf<int32_t> dg;
    DevBuf<IterState> st;
    xd.ensure(3 * m);
    yd.ensure(3 * n);
    dp.ensure(static_cast<size_t>(m) * n);
    dg.ensure(m);
    st.ensure(1);
    IterState h{};
    h.sigma2 = sigma2;
    h.sigma2_e_last = std::max(sigma2, kSigma2Floor);  // correspondence.hpp:43-47
    FCPD_CUDA(cudaMemcpyAsync(xd.p, xt, sizeof(double) * d * m, cudaMemcpyHostToDevice, str));
    FCPD_CUDA(cudaMemcpyAsync(yd.p, y, sizeof(double) * d * n, cudaMemcpyHostToDevice, str));
    FCPD_CUDA(cudaMemcpyAsync(st.p, &h, sizeof h, cudaMemcpyHostToDevice, str));
    FCPD_CUDA(cudaMemsetAsync(dg.p, 0, sizeof(int32_t) * m, str));
    launch_dense_posterior(xd.p, m, yd.p, n, d, omega, st.p, row_constrain, dg.p, dp.p, str);
    FCPD_CUDA(cudaMemcpyAsync(p, dp.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaMemcpyAsync(deg.data(), dg.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, str));
    FCPD_CUDA(cudaStreamSynchronize(str));
    if (clamped) *clamped = sigma2 < kSigma2Floor ? 1 : 0;
    for (auto* b : {&xd, &yd, &dp}) b->release();
    dg.release();
    st.release();
    int64_t nd = 0;
    if (row_constrain)
      for (int64_t i = 0; i < m; ++i)
        if (deg[i]) {
          if (degenerate_rows) degenerate_rows[nd] = i;
          ++nd;
        }
    if (n_degenerate) *n_degenerate = nd;
  });
}

int fcpd_build_gram(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d, double beta,
                    double* phi) {
  return guarded(ctx, [&] {
    if (m <= 0 || m > 46000) throw Failure(FCPD_ERR_PARAMETER, "build_gram: M out of range for the dense path");
    DevBuf<double> xd, g;
    xd.ensure(static_cast<size_t>(d) * m);
    g.ensure(static_cast<size_t>(m) * m);
    FCPD_CUDA(cudaMemcpyAsync(xd.p, x, sizeof(double) * d * m, cudaMemcpyHostToDevice, ctx->stream));
    build_gram_device(xd.p, m, d, beta, g.p, m, ctx->stream);
    FCPD_CUDA(cudaMemcpyAsync(phi, g.p, sizeof(double) * m * m, cudaMemcpyDeviceToHost, ctx->stream));
    FCPD_CUDA(cudaStreamSynchronize(ctx->stream));
    xd.release();
    g.release();
  });
}

int fcpd_build_basis(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d, double beta,
                     int64_t rank, double* u, double* lambda, double* lambda_raw) {
  return guarded(ctx, [&] {
    if (m <= 0 || m > 46000) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: M out of range for the dense path");
    if (rank < 1 || rank > m) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: rank out of [1, M]");
    DevBuf<double> xd, g;
    xd.ensure(static_cast<size_t>(d) * m);
    g.ensure(static_cast<size_t>(m) * m);
    FCPD_CUDA(cudaMemcpyAsync(xd.p, x, sizeof(double) * d * m, cudaMemcpyHostToDevice, ctx->stream));
    build_gram_device(xd.p, m, d, beta, g.p, m, ctx->stream);
    Basis b;
    dense_eigensolve(ctx->solver, g.p, m, rank, b, u, ctx->stream);
    if (lambda) std::copy(b.lam_host.begin(), b.lam_host.end(), lambda);
    if (lambda_raw) std::copy(b.lam_raw_host.begin(), b.lam_raw_host.end(), lambda_raw);
    b.release();
    xd.release();
    g.release();
  });
}

// ---- spectral cache (kernel.hpp:85-144): "FCPD", u32 version 1, u64 M,
// u64 K, f64 beta, U row-major f64 (M×K), λ f64 (K) — little-endian.

int fcpd_save_spectral_cache(fcpd_ctx* ctx, const char* path) {
  return guarded(ctx, [&] {
    Basis& b = ctx->basis;
    if (!b.u64 || b.m == 0) throw Failure(FCPD_ERR_PARAMETER, "spectral cache: no basis in context");
    std::vector<double> u(static_cast<size_t>(b.m * b.k));
    FCPD_CUDA(cudaMemcpyAsync(u.data(), b.u64, sizeof(double) * u.size(), cudaMemcpyDeviceToHost,
                              ctx->stream));
    FCPD_CUDA(cudaStreamSynchronize(ctx->stream));
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Failure(FCPD_ERR_IO, std::string("cannot open spectral cache for writing: ") + path);
    const uint32_t ver = 1;
    const uint64_t mm = static_cast<uint64_t>(b.m), kk = static_cast<uint64_t>(b.k);
    bool ok = std::fwrite("FCPD", 1, 4, f) == 4 && std::fwrite(&ver, 4, 1, f) == 1 &&
              std::fwrite(&mm, 8, 1, f) == 1 && std::fwrite(&kk, 8, 1, f) == 1 &&
              std::fwrite(&b.key_beta, 8, 1, f) == 1;
    // rows in the caller's point order (the device keeps them spatially sorted)
    std::vector<int64_t> inv(b.m);
    for (int64_t k = 0; k < b.m; ++k) inv[b.perm.empty() ? k : b.perm[k]] = k;
    std::vector<double> row(b.k);
    for (int64_t i = 0; ok && i < b.m; ++i) {
      for (int64_t j = 0; j < b.k; ++j) row[j] = u[j * b.m + inv[i]];
      ok = std::fwrite(row.data(), 8, b.k, f) == static_cast<size_t>(b.k);
    }
    ok = ok && std::fwrite(b.lam_host.data(), 8, b.k, f) == static_cast<size_t>(b.k);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw Failure(FCPD_ERR_IO, std::string("spectral cache write failed: ") + path);
  });
}

int fcpd_load_spectral_cache(fcpd_ctx* ctx, const char* path, const double* x, int64_t m,
                             const double* y, int64_t n, int32_t d, const fcpd_config* cfg) {
  return guarded(ctx, [&] {
    if (!cfg) throw Failure(FCPD_ERR_PARAMETER, "spectral cache: null config");
    validate_register(x, m, y, n, d, *cfg);
    FILE* f = std::fopen(path, "rb");
    if (!f) throw Failure(FCPD_ERR_IO, std::string("cannot open spectral cache: ") + path);
    char magic[4];
    uint32_t ver = 0;
    uint64_t mm = 0, kk = 0;
    double beta = 0.0;
    const bool hdr = std::fread(magic, 1, 4, f) == 4 && std::fread(&ver, 4, 1, f) == 1 &&
                     std::fread(&mm, 8, 1, f) == 1 && std::fread(&kk, 8, 1, f) == 1 &&
                     std::fread(&beta, 8, 1, f) == 1;
    if (!hdr || std::memcmp(magic, "FCPD", 4) != 0) {
      std::fclose(f);
      throw Failure(FCPD_ERR_PARSE, std::string("not a spectral cache file: ") + path);
    }
    if (ver != 1) {
      std::fclose(f);
      throw Failure(FCPD_ERR_PARSE, std::string("unsupported spectral cache version in ") + path);
    }
    const bool lowrank = cfg->variant == FCPD_VARIANT_FAST_LOWRANK;
    const int64_t rank = lowrank ? lowrank_rank(cfg->rank_fraction, m) : m;
    if (static_cast<int64_t>(mm) != m || static_cast<int64_t>(kk) != rank || beta != cfg->beta) {
      std::fclose(f);
      throw Failure(FCPD_ERR_PARAMETER, "spectral cache does not match (M, rank, beta) of the call");
    }
    std::vector<double> u(static_cast<size_t>(m * rank)), row(rank), lam(rank);
    bool ok = true;
    for (int64_t i = 0; ok && i < m; ++i) {
      ok = std::fread(row.data(), 8, rank, f) == static_cast<size_t>(rank);
      for (int64_t j = 0; j < rank; ++j) u[j * m + i] = row[j];
    }
    ok = ok && std::fread(lam.data(), 8, rank, f) == static_cast<size_t>(rank);
    std::fclose(f);
    if (!ok) throw Failure(FCPD_ERR_PARSE, std::string("truncated spectral cache: ") + path);
    // install under the key register_pointsets will compute for (x, y, cfg)
    std::vector<double> xs, ys;
    double center[3], scale;
    normalize_pair_host(x, m, y, n, d, cfg->normalize != 0, xs, ys, center, &scale);
    std::vector<int64_t> perm = spatial_sort(xs, m);  // the order register will use
    uint64_t h = fnv1a(xs.data(), sizeof(double) * xs.size());
    h = fnv1a(&m, sizeof m, h);
    h = fnv1a(&rank, sizeof rank, h);
    std::vector<double> us(u.size());
    for (int64_t j = 0; j < rank; ++j)
      for (int64_t k = 0; k < m; ++k) us[j * m + k] = u[j * m + perm[k]];
    Basis& b = ctx->basis;
    basis_from_host(b, us.data(), lam.data(), m, rank, ctx->stream);
    b.perm = perm;
    upload_lambda(b, !lowrank, ctx->stream);  // cached λ are the clamped ones
    b.key_hash = h;
    b.key_beta = cfg->beta;
    b.key_variant = cfg->variant;
  });
}

int fcpd_build_basis_topk(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d, double beta,
                          int64_t rank, int32_t iterations, double* u, double* lambda,
                          double* lambda_raw) {
  return guarded(ctx, [&] {
    if (m <= 0) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: empty point set");
    if (d < 1 || d > 3) throw Failure(FCPD_ERR_DIMENSION, "eigendecompose: the B200 path supports D <= 3");
    DevBuf<double> xd;
    xd.ensure(3 * static_cast<size_t>(m));
    FCPD_CUDA(cudaMemsetAsync(xd.p, 0, sizeof(double) * 3 * m, ctx->stream));
    FCPD_CUDA(cudaMemcpyAsync(xd.p, x, sizeof(double) * d * m, cudaMemcpyHostToDevice, ctx->stream));
    Basis b;
    topk_eigensolve(ctx->solver, ctx->blas, xd.p, m, d, beta, rank,
                    iterations > 0 ? iterations : topk_iterations(),
                    iterations <= 0 && topk_adaptive(), 0, b, ctx->stream, u);
    if (lambda) std::copy(b.lam_host.begin(), b.lam_host.end(), lambda);
    if (lambda_raw) std::copy(b.lam_raw_host.begin(), b.lam_raw_host.end(), lambda_raw);
    b.release();
    xd.release();
  });
}

// normalize_pair (pointset.hpp:124-148): host fp64, O(M+N) — the engine's
// own normalisation (normalize_pair_host), plus the reference's checks and
// degenerate flag.
int fcpd_normalize_pair(fcpd_ctx* ctx, const double* x, int64_t m, int32_t dx, const double* y,
                        int64_t n, int32_t dy, double* xo, double* yo, double* center,
                        double* scale, int32_t* degenerate) {
  return guarded(ctx, [&] {
    if (m <= 0 || n <= 0) throw Failure(FCPD_ERR_PARAMETER, "normalize_pair: empty point set");
    if (dx != dy) throw Failure(FCPD_ERR_DIMENSION, "normalize_pair: dimension mismatch");
    const int d = dx;
    const double total = static_cast<double>(m + n);
    std::vector<double> c(static_cast<size_t>(std::max(d, 1)), 0.0);
    for (int k = 0; k < d; ++k) {
      double sx = 0.0, sy = 0.0;
      for (int64_t i = 0; i < m; ++i) sx += x[k * m + i];
      for (int64_t i = 0; i < n; ++i) sy += y[k * n + i];
      c[k] = (sx + sy) / total;
    }
    double sc = 0.0;
    for (int k = 0; k < d; ++k) {
      for (int64_t i = 0; i < m; ++i) sc = std::max(sc, std::fabs(x[k * m + i] - c[k]));
      for (int64_t i = 0; i < n; ++i) sc = std::max(sc, std::fabs(y[k * n + i] - c[k]));
    }
    const bool deg = !(sc > 0.0);
    if (deg) sc = 1.0;
    for (int k = 0; k < d; ++k) {
      for (int64_t i = 0; i < m; ++i) xo[k * m + i] = (x[k * m + i] - c[k]) / sc;
      for (int64_t i = 0; i < n; ++i) yo[k * n + i] = (y[k * n + i] - c[k]) / sc;
      if (center) center[k] = c[k];
    }
    if (scale) *scale = sc;
    if (degenerate) *degenerate = deg ? 1 : 0;
  });
}

}  // extern "C"
