/* fcpd_capi.h — C ABI of the B200-native Fast-CPD engine (libfcpd_b200.so).
 *
 * This is the drop-in boundary for the reference's registration API
 * (/root/reference/proj/include/fastcpd/).  Plain pointers and sizes only; no
 * CUDA, Eigen or torch types.  All point sets are column-major (SoA) fp64
 * exactly like Eigen::MatrixXd (pointset.hpp:19-27): coordinate d of point i
 * lives at ptr[d*count + i].  Matrices such as the correspondence P are
 * column-major M×N.  Buffers are caller-owned host memory; every call copies
 * in and out once.
 *
 * Errors: every entry point returns FCPD_OK or one of the FCPD_ERR_* codes,
 * which map 1:1 to the reference exception hierarchy (errors.hpp:8-34);
 * fcpd_last_error() returns the message the reference would have thrown
 * (e.g. "register: iteration 3: update_sigma2: negative variance ...").
 * include/fastcpd/fastcpd.hpp rethrows them as fastcpd::ParameterError etc.
 *
 * Threading: one context per host thread; a context is not thread-safe.
 */
#ifndef FCPD_CAPI_H_
#define FCPD_CAPI_H_

#include <stdint.h>

#if defined(__GNUC__)
#define FCPD_API __attribute__((visibility("default")))
#else
#define FCPD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* error codes — errors.hpp:8-34 */
#define FCPD_OK 0
#define FCPD_ERR_PARAMETER 1 /* ParameterError */
#define FCPD_ERR_DIMENSION 2 /* DimensionError */
#define FCPD_ERR_NUMERIC 3   /* NumericError */
#define FCPD_ERR_IO 4        /* IoError */
#define FCPD_ERR_PARSE 5     /* ParseError */
#define FCPD_ERR_CUDA 10     /* CUDA runtime / cuSOLVER failure */
#define FCPD_ERR_NCCL 11     /* NCCL failure (multi-GPU) */
#define FCPD_ERR_OOM 12      /* device allocation failed */

/* SolverVariant — solvers.hpp:18.  Only the fast variants run on the device
 * (the north-star path); cpd / cpd_lowrank return FCPD_ERR_PARAMETER. */
#define FCPD_VARIANT_CPD 0
#define FCPD_VARIANT_CPD_LOWRANK 1
#define FCPD_VARIANT_FAST 2
#define FCPD_VARIANT_FAST_LOWRANK 3

/* RegistrationConfig — registration.hpp:30-40 (same fields, same defaults
 * via fcpd_config_default). */
typedef struct fcpd_config {
  double omega;         /* uniform outlier weight, [0,1)          (0.7)  */
  double beta;          /* Gaussian kernel width                  (2.0)  */
  double lambda_reg;    /* regularisation λ                       (10.0) */
  int32_t iterations;   /* fixed EM iteration count               (100)  */
  int32_t variant;      /* FCPD_VARIANT_*                         (fast) */
  double rank_fraction; /* K = llround(rank_fraction·M), low rank (0.1)  */
  uint64_t seed;        /* echoed only, as in the reference       (0)    */
  int32_t normalize;    /* normalize_pair before registering      (1)    */
  int32_t early_stop;   /* stop when |Δσ²| < 1e-10                 (0)    */
  int32_t pad0;
  double spectral_tau;  /* extension: the basis streams skip eigenpairs
                           whose filter λnum/(λ+λ_reg σ²) < tau; their
                           contribution to x̃ is far below the fp32 basis
                           rounding (1e-10; 0 = stream all K)             */
} fcpd_config;

/* TimingBreakdown — registration.hpp:21-28, plus t_setup (Gram build +
 * eigendecomposition, reported separately; the reference folds the Gram
 * build into t_o).  Identities t_f = t_eig + t_iter and
 * t_total = t_c + t_f + t_o hold exactly.  In-loop phases are measured on
 * the device (%globaltimer at kernel boundaries). */
typedef struct fcpd_timing {
  double t_c, t_eig, t_iter, t_f, t_o, t_total;
  double t_setup;
} fcpd_timing;

/* RegistrationResult — registration.hpp:48-56.  Null pointers skip that
 * output.  `correspondence` (M×N column-major, the final row-constrained P̃)
 * is materialised only when non-null; the hot path never forms it. */
typedef struct fcpd_result {
  double* transformed;      /* M×D, original units when normalize   */
  double* coefficients;     /* M×D, W of the last iteration          */
  double* sigma2_trace;     /* capacity cfg.iterations               */
  double* correspondence;   /* optional M×N                          */
  int32_t* degenerate_mask; /* optional M: last E-step's uniform rows */
  int32_t iterations_run;
  int32_t basis_reused;     /* 1 if the cached spectral basis was used */
  double sigma2_initial;
  int64_t degenerate_rows;  /* RegistrationDiagnostics — cumulative   */
  int64_t sigma2_clamps;
  fcpd_timing timing;
  int64_t h2d_bytes;        /* host→device bytes this call copied     */
  int64_t d2h_bytes;        /* device→host bytes this call copied     */
  int64_t tiles_evaluated[2]; /* E-step (256-point block, 32-point
                                 sub-tile) pairs computed since the
                                 session began (pass 1: scene blocks ×
                                 model sub-tiles; pass 2: model blocks ×
                                 scene sub-tiles); the rest were culled
                                 (≤ 2^-32 of any total)                 */
  int64_t spectral_rank;    /* eigenpairs the last iteration's basis
                               streams used (filter ≥ tau; = K untruncated) */
  int32_t mstep_fused;      /* 1 if the session ran the one-kernel M-step */
  int32_t reserved0;
  int64_t pairs_by_form[4]; /* E-step (m, n) pair slots evaluated since the
                               session began, by (pass 1 centred, pass 1
                               difference, pass 2 centred, pass 2
                               difference) pair form — the instruction mix
                               the E-step roofline is computed from (culling
                               sessions; 0 otherwise)                    */
} fcpd_result;

typedef struct fcpd_ctx fcpd_ctx;

/* Default config (registration.hpp:30-40). */
FCPD_API void fcpd_config_default(fcpd_config* cfg);

/* Context: binds one CUDA device (its own stream, cuSOLVER handle, cached
 * spectral basis and CUDA graphs). */
FCPD_API int fcpd_create(fcpd_ctx** out, int device);
FCPD_API void fcpd_destroy(fcpd_ctx* ctx);
FCPD_API const char* fcpd_last_error(const fcpd_ctx* ctx);
FCPD_API const char* fcpd_version(void);

/* Multi-GPU (one process per GPU): rank 0 calls fcpd_nccl_unique_id and
 * shares the 128 bytes with the other ranks (e.g. torch.distributed); each
 * rank then creates its context with fcpd_create_dist.  In such a context
 * fcpd_register / fcpd_session_begin take the FULL model x and this rank's
 * SHARD of the scene y (n = local count); the scene is reduced over ranks,
 * the model rows and the basis are row-sharded, and every
 * rank receives the full result.  Correspondence output is single-GPU only. */
FCPD_API int fcpd_nccl_unique_id(uint8_t* out128);
FCPD_API int fcpd_create_dist(fcpd_ctx** out, int device, int rank, int world,
                              const uint8_t* id128);
FCPD_API int fcpd_world(const fcpd_ctx* ctx, int32_t* rank, int32_t* world);
/* A loopback group: `world` (≤ 8) virtual ranks on ONE device driven by one
 * context — the scene-sharded data plane of fcpd_create_dist with the
 * collectives as device kernels, for testing the multi-rank path on one GPU.
 * fcpd_register / fcpd_session_begin on it take the FULL scene (split into
 * `world` contiguous shards, rows [r·N/world, (r+1)·N/world)). */
FCPD_API int fcpd_create_loopback(fcpd_ctx** out, int device, int world);

/* register_pointsets — registration.hpp:79-175.  x: M×D model, y: N×D scene.
 * The spectral basis is cached in the context keyed by (normalised X, β,
 * rank); a repeated call on the same model reuses it (the paper's
 * "precomputed in advance" protocol) and reports t_eig = 0. */
FCPD_API int fcpd_register(fcpd_ctx* ctx, const double* x, int64_t m, const double* y, int64_t n,
                  int32_t d, const fcpd_config* cfg, fcpd_result* out);

/* Device-resident session (bench / serving): inputs copied once, then EM
 * iterations are replayed from a CUDA graph without host round trips. */
FCPD_API int fcpd_session_begin(fcpd_ctx* ctx, const double* x, int64_t m, const double* y,
                       int64_t n, int32_t d, const fcpd_config* cfg);
FCPD_API int fcpd_session_run(fcpd_ctx* ctx, int32_t iterations); /* async on the ctx stream */
FCPD_API int fcpd_session_sync(fcpd_ctx* ctx);
FCPD_API int fcpd_session_read(fcpd_ctx* ctx, fcpd_result* out);
/* Eager profiling of `iterations` more session iterations with CUDA events
 * between kernel groups on the context stream.  ms_per_phase[6] receives the
 * mean ms of: E pass 1 (column normalisers), E pass 2 (row accumulation),
 * Qᵀ·R stream, z-reduce/filter, Q·g stream, transform + σ². */
FCPD_API int fcpd_session_profile(fcpd_ctx* ctx, int32_t iterations, double* ms_per_phase);
/* The cudaStream_t the context launches on, as an opaque pointer. */
FCPD_API void* fcpd_stream(fcpd_ctx* ctx);
/* Number of kernels one EM iteration launches (the graph's kernel nodes). */
FCPD_API int32_t fcpd_kernels_per_iteration(const fcpd_ctx* ctx);

/* ---- fine-grained entry points (the reference's L2 functions) ---------- */

/* posterior + enforce_row_constraint + estimated_targets —
 * correspondence.hpp:35-105 — without forming P.  Outputs per model row:
 * ptilde_y (M×D) = (P̃Y)_m, p1 (M) = raw row mass Σ_n P_mn, var (M) =
 * Σ_n P̃_mn‖y_n−x_m‖², degenerate (M) = uniform-row flag; per scene column
 * pt1 (N) = Σ_m P_mn.  Any output may be null.  `clamped` receives
 * Correspondence::sigma2_clamped. */
FCPD_API int fcpd_estep(fcpd_ctx* ctx, const double* xt, int64_t m, const double* y, int64_t n,
               int32_t d, double omega, double sigma2, double* ptilde_y, double* p1,
               double* var, int32_t* degenerate, double* pt1, int32_t* clamped);

/* posterior (correspondence.hpp:35-79), materialised M×N on the device;
 * if row_constrain, also enforce_row_constraint (:83-98) and the degenerate
 * row list (capacity M).  For small problems and tests. */
FCPD_API int fcpd_posterior_dense(fcpd_ctx* ctx, const double* xt, int64_t m, const double* y,
                         int64_t n, int32_t d, double omega, double sigma2, int32_t row_constrain,
                         double* p, int32_t* clamped, int64_t* degenerate_rows,
                         int64_t* n_degenerate);

/* build_gram + eigendecompose — kernel.hpp:31-72 — on the device in fp64:
 * u (M×rank column-major), lambda (clamped, descending), lambda_raw. */
FCPD_API int fcpd_build_basis(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d, double beta,
                     int64_t rank, double* u, double* lambda, double* lambda_raw);

/* Top-K eigenpairs of Φ without forming it (configs 2–4): randomized block
 * subspace iteration with on-the-fly fp64 Φ·V products + Rayleigh–Ritz,
 * `iterations` power steps; 0 → up to 4, stopping once every top-K Ritz
 * residual ‖Φu − θu‖ ≤ 1e-11·θ₁.  Same outputs and clamp as
 * fcpd_build_basis. */
FCPD_API int fcpd_build_basis_topk(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d,
                                   double beta, int64_t rank, int32_t iterations, double* u,
                                   double* lambda, double* lambda_raw);

/* Spectral cache — kernel.hpp:85-144, the reference's binary format ("FCPD",
 * u32 version 1, u64 M, u64 K, f64 beta, U row-major f64, λ f64).  save
 * writes the context's current basis (the one the last register/session
 * built or reused); load installs a cached basis for the model of the
 * (x, y, cfg) call (normalised exactly as fcpd_register will) so the next
 * fcpd_register on them skips the eigensolve (the paper's precomputed
 * basis).  Mismatched (M, rank, β) → FCPD_ERR_PARAMETER. */
FCPD_API int fcpd_save_spectral_cache(fcpd_ctx* ctx, const char* path);
FCPD_API int fcpd_load_spectral_cache(fcpd_ctx* ctx, const char* path, const double* x,
                                      int64_t m, const double* y, int64_t n, int32_t d,
                                      const fcpd_config* cfg);

/* build_gram — kernel.hpp:31-47 — M×M column-major fp64. */
FCPD_API int fcpd_build_gram(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d, double beta,
                    double* phi);

/* ---- the reference's L2 functions in fp64 on the device (l2api.cu) -------
 * Same semantics, checks and messages as the reference functions named;
 * dense inputs as the caller passes them (column-major), products through
 * cuBLAS dgemm, fixed-order reductions.  For the reference's unit tests and
 * drop-in callers of these functions — the EM hot path (fcpd_register) does
 * not use them. */

/* estimated_targets — correspondence.hpp:101-105: out (M×D) = P (M×N) · Y
 * (NY×D); NY != N → FCPD_ERR_PARAMETER "estimated_targets: shape mismatch". */
FCPD_API int fcpd_estimated_targets(fcpd_ctx* ctx, const double* p, int64_t m, int64_t n,
                                    const double* y, int64_t ny, int32_t d, double* out);

/* enforce_row_constraint — correspondence.hpp:83-98, in place on P (M×N):
 * rows with sum < 1e-300 become 1/N (degenerate[i] = 1), others / sum. */
FCPD_API int fcpd_enforce_row_constraint(fcpd_ctx* ctx, double* p, int64_t m, int64_t n,
                                         int32_t* degenerate);

/* update_sigma2 — solvers.hpp:160-176 (trace form): y N×D, P M×NP, x̃ MX×D.
 * !row_constrained → FCPD_ERR_PARAMETER; value < −1e-8 → FCPD_ERR_NUMERIC;
 * *out = max(value, 1e-10). */
FCPD_API int fcpd_update_sigma2(fcpd_ctx* ctx, const double* y, int64_t n, const double* p,
                                int64_t m, int64_t np, const double* xt, int64_t mx, int32_t d,
                                int32_t row_constrained, double* out);

/* eigendecompose — kernel.hpp:49-72 — of a given Φ (M×M): top `rank`
 * eigenpairs, descending, 1e-12·λmax clamp (lambda) and raw (lambda_raw). */
FCPD_API int fcpd_eigendecompose(fcpd_ctx* ctx, const double* phi, int64_t m, int64_t rank,
                                 double* u, double* lambda, double* lambda_raw);

/* solve_fast_lowrank — solvers.hpp:61-73: W (M×D) = U diag(1/(λ+λ_reg σ²))
 * Uᵀ R; u M×K, residual RM×D (RM != M → FCPD_ERR_PARAMETER); a non-positive
 * λ_i + λ_reg σ² → FCPD_ERR_NUMERIC.  solve_fast (:75-80) is K = M. */
FCPD_API int fcpd_solve_fast_lowrank(fcpd_ctx* ctx, const double* u, const double* lambda,
                                     int64_t m, int64_t k, double lambda_reg, double sigma2,
                                     const double* residual, int64_t rm, int32_t d, double* w);

/* apply_transform — solvers.hpp:138-144: out = X + Φ W (Φ MPHI×MPHI, W
 * MW×DW; any mismatch with X (M×D) → "apply_transform: shape mismatch"). */
FCPD_API int fcpd_apply_transform(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d,
                                  const double* phi, int64_t mphi, const double* w, int64_t mw,
                                  int32_t dw, double* out);

/* apply_transform_lowrank — solvers.hpp:147-155: out = X + U Λ Uᵀ W. */
FCPD_API int fcpd_apply_transform_lowrank(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d,
                                          const double* u, int64_t mu, const double* lambda,
                                          int64_t k, const double* w, int64_t mw, int32_t dw,
                                          double* out);

/* lowrank_reconstruction_error — kernel.hpp:76-83: ‖Φ − U Λ Uᵀ‖_F. */
FCPD_API int fcpd_lowrank_reconstruction_error(fcpd_ctx* ctx, const double* phi, int64_t m,
                                               const double* u, int64_t mu,
                                               const double* lambda, int64_t k, double* out);

/* normalize_pair — pointset.hpp:124-148 (host fp64): joint centroid,
 * max-abs scale (≤ 0 → 1 and *degenerate = 1); xo/yo as x/y. */
FCPD_API int fcpd_normalize_pair(fcpd_ctx* ctx, const double* x, int64_t m, int32_t dx,
                                 const double* y, int64_t n, int32_t dy, double* xo, double* yo,
                                 double* center, double* scale, int32_t* degenerate);

#ifdef __cplusplus
}
#endif
#endif /* FCPD_CAPI_H_ */
