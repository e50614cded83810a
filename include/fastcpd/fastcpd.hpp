// fastcpd/fastcpd.hpp — drop-in C++ API for the B200 engine.
//
// Mirrors the reference's public headers (proj/include/fastcpd/*.hpp) for the
// registration path: the same namespace, type names, field names, defaults
// and exception classes, so code written against
//   fastcpd::register_pointsets(const PointSet&, const PointSet&,
//                               const RegistrationConfig&)
// (registration.hpp:79-81) compiles against this header and runs on the GPU
// through the C ABI in fcpd_capi.h.  Differences:
//  * PointSet::pts is fastcpd::Matrix (column-major, Eigen-compatible layout
//    and the Eigen accessors used by the reference's callers: rows(), cols(),
//    operator()(i,j), data(), resize(), setZero()).  Define
//    FASTCPD_USE_EIGEN before including to use Eigen::MatrixXd instead.
//  * RegistrationResult::correspondence is filled only when
//    cfg.want_correspondence is set (the device path never forms the M×N P).
//  * Only the fast / fast_lowrank variants run on the device; cpd variants
//    throw ParameterError (they are the reference's O(M³) baselines).
#pragma once

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "fcpd_capi.h"

#ifdef FASTCPD_USE_EIGEN
#include <Eigen/Core>
#endif

namespace fastcpd {

// ------------------------------------------------------ errors.hpp:8-34
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : Error {
  using Error::Error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct ParameterError : Error {
  using Error::Error;
};
struct NumericError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};
struct DeviceError : Error {  // CUDA / NCCL / out of device memory
  using Error::Error;
};

inline void throw_code(int code, const std::string& msg) {
  switch (code) {
    case FCPD_OK: return;
    case FCPD_ERR_PARAMETER: throw ParameterError(msg);
    case FCPD_ERR_DIMENSION: throw DimensionError(msg);
    case FCPD_ERR_NUMERIC: throw NumericError(msg);
    case FCPD_ERR_IO: throw IoError(msg);
    case FCPD_ERR_PARSE: throw ParseError(msg);
    default: throw DeviceError(msg);
  }
}

// -------------------------------------------------------------- matrix
#ifdef FASTCPD_USE_EIGEN
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;
// Column-major dense fp64 matrix: the subset of Eigen::MatrixXd the
// registration API and its callers use.
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(j * r_ + i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    v_.assign(static_cast<size_t>(r * c), 0.0);
  }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

// fp64 vector: the subset of Eigen::VectorXd the L2 types use.
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  Index size() const { return static_cast<Index>(v_.size()); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
  double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }

 private:
  std::vector<double> v_;
};
#endif

// -------------------------------------------------- pointset.hpp:19-43
struct PointSet {
  Matrix pts;
  PointSet() = default;
  explicit PointSet(Matrix p) : pts(std::move(p)) {}
  Index count() const { return pts.rows(); }
  Index dim() const { return pts.cols(); }
};

// ------------------------------------------------------ solvers.hpp:14-54
struct Coefficients {
  Matrix w;
};

enum class SolverVariant { cpd, cpd_lowrank, fast, fast_lowrank };

inline const char* to_string(SolverVariant v) {
  switch (v) {
    case SolverVariant::cpd: return "cpd";
    case SolverVariant::cpd_lowrank: return "cpd_lowrank";
    case SolverVariant::fast: return "fast";
    case SolverVariant::fast_lowrank: return "fast_lowrank";
  }
  return "?";
}

inline SolverVariant variant_from_string(const std::string& s) {
  if (s == "cpd") return SolverVariant::cpd;
  if (s == "cpd_lowrank" || s == "cpd-lowrank") return SolverVariant::cpd_lowrank;
  if (s == "fast") return SolverVariant::fast;
  if (s == "fast_lowrank" || s == "fast-lowrank") return SolverVariant::fast_lowrank;
  throw ParameterError("unknown solver variant: " + s);
}

inline bool is_lowrank(SolverVariant v) {
  return v == SolverVariant::cpd_lowrank || v == SolverVariant::fast_lowrank;
}
inline bool is_fast(SolverVariant v) {
  return v == SolverVariant::fast || v == SolverVariant::fast_lowrank;
}

inline Index lowrank_rank(double rank_fraction, Index m) {
  if (rank_fraction <= 0.0 || rank_fraction > 1.0)
    throw ParameterError("rank_fraction must lie in (0, 1]");
  Index k = static_cast<Index>(std::llround(rank_fraction * static_cast<double>(m)));
  if (k < 1) k = 1;
  if (k > m) k = m;
  return k;
}

// --------------------------------------------- correspondence.hpp:12-29
inline constexpr double kSigma2Floor = 1e-10;

struct Correspondence {
  Matrix p;
  bool row_constrained = false;
  std::vector<Index> degenerate_rows;
  bool sigma2_clamped = false;

  Vector row_sums() const {
    Vector s(p.rows());
    for (Index j = 0; j < p.cols(); ++j)
      for (Index i = 0; i < p.rows(); ++i) s(i) += p(i, j);
    return s;
  }
  Vector col_sums() const {
    Vector s(p.cols());
    for (Index j = 0; j < p.cols(); ++j)
      for (Index i = 0; i < p.rows(); ++i) s(j) += p(i, j);
    return s;
  }
};

// ------------------------------------------------ registration.hpp:21-56
struct TimingBreakdown {
  double t_c = 0.0, t_eig = 0.0, t_iter = 0.0, t_f = 0.0, t_o = 0.0, t_total = 0.0;
  double t_setup = 0.0;  // extension: Gram build + eigendecomposition
};

struct RegistrationConfig {
  double omega = 0.7;
  double beta = 2.0;
  double lambda_reg = 10.0;
  int iterations = 100;
  SolverVariant variant = SolverVariant::fast;
  double rank_fraction = 0.1;
  unsigned long seed = 0;
  bool normalize = true;
  bool early_stop = false;
  bool want_correspondence = false;  // extension: materialise P̃ (M×N) at the end
  int device = 0;                    // extension: CUDA device of the default context
  double spectral_tau = 1e-10;       // extension: basis-stream filter threshold (0 = all K)
};

struct RegistrationDiagnostics {
  long degenerate_rows = 0;
  long sigma2_clamps = 0;
  std::string baseline_solver = "dense LDLT factorization";
};

struct RegistrationResult {
  PointSet transformed;
  Coefficients coefficients;
  Correspondence correspondence;
  std::vector<double> sigma2_trace;
  TimingBreakdown timing;
  RegistrationDiagnostics diagnostics;
  double sigma2_initial = 0.0;
};

// ----------------------------------------------------------- context
// One engine context per device per thread (stream, cuSOLVER handle, cached
// spectral basis).  register_pointsets() uses a thread-local default.
class Context {
 public:
  explicit Context(int device = 0) {
    fcpd_ctx* c = nullptr;
    const int rc = fcpd_create(&c, device);
    if (rc != FCPD_OK) throw_code(rc, "fcpd_create failed on device " + std::to_string(device));
    ctx_.reset(c);
  }
  fcpd_ctx* get() const { return ctx_.get(); }
  void check(int rc) const {
    if (rc != FCPD_OK) throw_code(rc, fcpd_last_error(ctx_.get()));
  }

  RegistrationResult register_pointsets(const PointSet& x, const PointSet& y,
                                        const RegistrationConfig& cfg) const {
    if (x.count() == 0 || y.count() == 0) throw ParameterError("register: empty point set");
    if (x.dim() != y.dim()) throw DimensionError("register: model and scene dimension mismatch");
    const Index m = x.count(), n = y.count(), d = x.dim();
    fcpd_config c;
    fcpd_config_default(&c);
    c.omega = cfg.omega;
    c.beta = cfg.beta;
    c.lambda_reg = cfg.lambda_reg;
    c.iterations = cfg.iterations;
    c.variant = static_cast<int32_t>(cfg.variant);
    c.rank_fraction = cfg.rank_fraction;
    c.seed = cfg.seed;
    c.normalize = cfg.normalize ? 1 : 0;
    c.early_stop = cfg.early_stop ? 1 : 0;
    c.spectral_tau = cfg.spectral_tau;
    RegistrationResult res;
    res.transformed.pts.resize(m, d);
    res.coefficients.w.resize(m, d);
    res.sigma2_trace.assign(static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 1), 0.0);
    std::vector<int32_t> mask(static_cast<size_t>(m), 0);
    fcpd_result out{};
    out.transformed = res.transformed.pts.data();
    out.coefficients = res.coefficients.w.data();
    out.sigma2_trace = res.sigma2_trace.data();
    out.degenerate_mask = mask.data();
    if (cfg.want_correspondence) {
      res.correspondence.p.resize(m, n);
      out.correspondence = res.correspondence.p.data();
    }
    check(fcpd_register(ctx_.get(), x.pts.data(), m, y.pts.data(), n, static_cast<int32_t>(d),
                        &c, &out));
    res.sigma2_trace.resize(static_cast<size_t>(out.iterations_run));
    res.sigma2_initial = out.sigma2_initial;
    res.diagnostics.degenerate_rows = static_cast<long>(out.degenerate_rows);
    res.diagnostics.sigma2_clamps = static_cast<long>(out.sigma2_clamps);
    res.timing = TimingBreakdown{out.timing.t_c,   out.timing.t_eig, out.timing.t_iter,
                                 out.timing.t_f,   out.timing.t_o,   out.timing.t_total,
                                 out.timing.t_setup};
    res.correspondence.row_constrained = out.iterations_run > 0;
    for (Index i = 0; i < m; ++i)
      if (mask[static_cast<size_t>(i)]) res.correspondence.degenerate_rows.push_back(i);
    return res;
  }

 private:
  struct Del {
    void operator()(fcpd_ctx* c) const { fcpd_destroy(c); }
  };
  std::unique_ptr<fcpd_ctx, Del> ctx_;
};

inline Context& default_context(int device = 0) {
  thread_local std::unique_ptr<Context> ctx;
  thread_local int dev = -1;
  if (!ctx || dev != device) {
    ctx = std::make_unique<Context>(device);
    dev = device;
  }
  return *ctx;
}

// registration.hpp:79-175 — the drop-in entry point.
inline RegistrationResult register_pointsets(const PointSet& x, const PointSet& y,
                                             const RegistrationConfig& cfg) {
  return default_context(cfg.device).register_pointsets(x, y, cfg);
}

// ============================================================ L2 functions
// The reference's numerics entry points (correspondence.hpp, kernel.hpp,
// solvers.hpp, pointset.hpp) with the same names, types, checks and
// exceptions, running in fp64 on the default context's device through the
// C ABI (fcpd_capi.h, l2api.cu).  register_pointsets does not call these:
// its EM loop is the fused device path.

// --------------------------------------------- correspondence.hpp:15-18
struct GmmParams {
  double omega = 0.7;   // uniform outlier weight, [0,1)
  double sigma2 = 1.0;  // shared isotropic variance
};

namespace detail {
inline fcpd_ctx* l2ctx() { return default_context().get(); }
inline void l2check(int rc) {
  if (rc != FCPD_OK) throw_code(rc, fcpd_last_error(l2ctx()));
}
}  // namespace detail

// correspondence.hpp:35-79 — GMM posterior with the per-column max shift
// (materialised M×N; the dense fp64 device kernel).
inline Correspondence posterior(const PointSet& x_t, const PointSet& y, const GmmParams& params) {
  if (params.omega < 0.0 || params.omega >= 1.0)
    throw ParameterError("posterior: omega must lie in [0, 1)");
  if (x_t.dim() != y.dim()) throw DimensionError("posterior: dimension mismatch");
  Correspondence c;
  c.p.resize(x_t.count(), y.count());
  int32_t clamped = 0;
  int64_t nd = 0;
  detail::l2check(fcpd_posterior_dense(detail::l2ctx(), x_t.pts.data(), x_t.count(), y.pts.data(),
                                       y.count(), static_cast<int32_t>(x_t.dim()), params.omega,
                                       params.sigma2, 0, c.p.data(), &clamped, nullptr, &nd));
  c.sigma2_clamped = clamped != 0;
  c.row_constrained = false;
  return c;
}

// correspondence.hpp:83-98 — row normalisation with the uniform fallback.
inline Correspondence enforce_row_constraint(const Correspondence& raw) {
  Correspondence out = raw;
  out.degenerate_rows.clear();
  std::vector<int32_t> deg(static_cast<size_t>(raw.p.rows()), 0);
  detail::l2check(fcpd_enforce_row_constraint(detail::l2ctx(), out.p.data(), out.p.rows(),
                                              out.p.cols(), deg.data()));
  for (Index i = 0; i < out.p.rows(); ++i)
    if (deg[static_cast<size_t>(i)]) out.degenerate_rows.push_back(i);
  out.row_constrained = true;
  return out;
}

// correspondence.hpp:101-105 — Ỹ = P·Y.
inline PointSet estimated_targets(const Correspondence& p, const PointSet& y) {
  if (p.p.cols() != y.count()) throw ParameterError("estimated_targets: shape mismatch");
  PointSet out;
  out.pts.resize(p.p.rows(), y.dim());
  detail::l2check(fcpd_estimated_targets(detail::l2ctx(), p.p.data(), p.p.rows(), p.p.cols(),
                                         y.pts.data(), y.count(), static_cast<int32_t>(y.dim()),
                                         out.pts.data()));
  return out;
}

// ------------------------------------------------------ kernel.hpp:15-29
struct GramKernel {
  Matrix phi;
  double beta = 0.0;
  Index size() const { return phi.rows(); }
};

struct SpectralBasis {
  Matrix u;       // M × K, orthonormal columns
  Vector lambda;  // K, descending
  Index points() const { return u.rows(); }
  Index rank() const { return u.cols(); }
};

// kernel.hpp:31-47 — Φ_ij = exp(−‖x_i − x_j‖²/2β²), symmetric, unit diagonal.
inline GramKernel build_gram(const PointSet& x, double beta) {
  if (beta <= 0.0) throw ParameterError("build_gram: beta must be positive");
  GramKernel k;
  k.beta = beta;
  k.phi.resize(x.count(), x.count());
  detail::l2check(fcpd_build_gram(detail::l2ctx(), x.pts.data(), x.count(),
                                  static_cast<int32_t>(x.dim()), beta, k.phi.data()));
  return k;
}

// kernel.hpp:49-72 — top `rank` eigenpairs (cuSOLVER syevd, fp64),
// descending, λ < 1e-12·λmax clamped to 0.
inline SpectralBasis eigendecompose(const GramKernel& k, Index rank) {
  const Index m = k.size();
  if (rank < 1 || rank > m) throw ParameterError("eigendecompose: rank out of [1, M]");
  SpectralBasis b;
  b.u.resize(m, rank);
  b.lambda.resize(rank);
  detail::l2check(fcpd_eigendecompose(detail::l2ctx(), k.phi.data(), m, rank, b.u.data(),
                                      b.lambda.data(), nullptr));
  return b;
}

// kernel.hpp:76-83 — ‖Φ − U Λ Uᵀ‖_F.
inline double lowrank_reconstruction_error(const SpectralBasis& b, const GramKernel& k) {
  if (b.points() != k.size())
    throw ParameterError("lowrank_reconstruction_error: size mismatch");
  double e = 0.0;
  detail::l2check(fcpd_lowrank_reconstruction_error(detail::l2ctx(), k.phi.data(), k.size(),
                                                    b.u.data(), b.points(), b.lambda.data(),
                                                    b.rank(), &e));
  return e;
}

// kernel.hpp:85-144 — the spectral cache file: "FCPD", u32 version 1, u64 M,
// u64 K, f64 β, then U row by row and λ, little-endian fp64 (host I/O).
inline void save_spectral_cache(const std::string& path, const SpectralBasis& b, double beta) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError("cannot open spectral cache for writing: " + path);
  const uint32_t version = 1;
  const uint64_t m = static_cast<uint64_t>(b.points()), k = static_cast<uint64_t>(b.rank());
  bool ok = std::fwrite("FCPD", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
            std::fwrite(&m, 8, 1, f) == 1 && std::fwrite(&k, 8, 1, f) == 1 &&
            std::fwrite(&beta, 8, 1, f) == 1;
  std::vector<double> row(static_cast<size_t>(k));
  for (uint64_t i = 0; ok && i < m; ++i) {
    for (uint64_t j = 0; j < k; ++j)
      row[static_cast<size_t>(j)] = b.u(static_cast<Index>(i), static_cast<Index>(j));
    ok = std::fwrite(row.data(), 8, static_cast<size_t>(k), f) == static_cast<size_t>(k);
  }
  ok = ok && std::fwrite(b.lambda.data(), 8, static_cast<size_t>(k), f) == static_cast<size_t>(k);
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw IoError("spectral cache write failed: " + path);
}

inline SpectralBasis load_spectral_cache(const std::string& path, double* beta_out = nullptr) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open spectral cache: " + path);
  char magic[4] = {0, 0, 0, 0};
  uint32_t version = 0;
  uint64_t m = 0, k = 0;
  double beta = 0.0;
  const bool head = std::fread(magic, 1, 4, f) == 4 && std::fread(&version, 4, 1, f) == 1 &&
                    std::fread(&m, 8, 1, f) == 1 && std::fread(&k, 8, 1, f) == 1 &&
                    std::fread(&beta, 8, 1, f) == 1;
  if (!head || std::string(magic, 4) != "FCPD") {
    std::fclose(f);
    throw ParseError("not a spectral cache file: " + path);
  }
  if (version != 1) {
    std::fclose(f);
    throw ParseError("unsupported spectral cache version in " + path);
  }
  SpectralBasis b;
  b.u.resize(static_cast<Index>(m), static_cast<Index>(k));
  b.lambda.resize(static_cast<Index>(k));
  std::vector<double> row(static_cast<size_t>(k));
  bool ok = true;
  for (uint64_t i = 0; ok && i < m; ++i) {
    ok = std::fread(row.data(), 8, static_cast<size_t>(k), f) == static_cast<size_t>(k);
    for (uint64_t j = 0; ok && j < k; ++j)
      b.u(static_cast<Index>(i), static_cast<Index>(j)) = row[static_cast<size_t>(j)];
  }
  ok = ok && std::fread(b.lambda.data(), 8, static_cast<size_t>(k), f) == static_cast<size_t>(k);
  std::fclose(f);
  if (!ok) throw ParseError("truncated spectral cache: " + path);
  if (beta_out) *beta_out = beta;
  return b;
}

// ----------------------------------------------------- solvers.hpp:61-176
// solvers.hpp:61-73 — W = U (Λ + λσ² I)⁻¹ Uᵀ R.
inline Coefficients solve_fast_lowrank(const SpectralBasis& basis, double lambda_reg,
                                       double sigma2, const Matrix& residual) {
  if (basis.points() != residual.rows())
    throw ParameterError("solve_fast: residual rows must match basis points");
  Coefficients c;
  c.w.resize(residual.rows(), residual.cols());
  detail::l2check(fcpd_solve_fast_lowrank(detail::l2ctx(), basis.u.data(), basis.lambda.data(),
                                          basis.points(), basis.rank(), lambda_reg, sigma2,
                                          residual.data(), residual.rows(),
                                          static_cast<int32_t>(residual.cols()), c.w.data()));
  return c;
}

// solvers.hpp:75-80.
inline Coefficients solve_fast(const SpectralBasis& basis, double lambda_reg, double sigma2,
                               const Matrix& residual) {
  if (basis.rank() != basis.points())
    throw ParameterError("solve_fast expects the full spectral basis");
  return solve_fast_lowrank(basis, lambda_reg, sigma2, residual);
}

// solvers.hpp:138-144 — X + Φ W.
inline PointSet apply_transform(const PointSet& x, const GramKernel& k, const Coefficients& c) {
  if (k.size() != x.count() || c.w.rows() != x.count() || c.w.cols() != x.dim())
    throw ParameterError("apply_transform: shape mismatch");
  PointSet out;
  out.pts.resize(x.count(), x.dim());
  detail::l2check(fcpd_apply_transform(detail::l2ctx(), x.pts.data(), x.count(),
                                       static_cast<int32_t>(x.dim()), k.phi.data(), k.size(),
                                       c.w.data(), c.w.rows(), static_cast<int32_t>(c.w.cols()),
                                       out.pts.data()));
  return out;
}

// solvers.hpp:147-155 — X + U Λ Uᵀ W.
inline PointSet apply_transform_lowrank(const PointSet& x, const SpectralBasis& basis,
                                        const Coefficients& c) {
  if (basis.points() != x.count() || c.w.rows() != x.count() || c.w.cols() != x.dim())
    throw ParameterError("apply_transform_lowrank: shape mismatch");
  PointSet out;
  out.pts.resize(x.count(), x.dim());
  detail::l2check(fcpd_apply_transform_lowrank(
      detail::l2ctx(), x.pts.data(), x.count(), static_cast<int32_t>(x.dim()), basis.u.data(),
      basis.points(), basis.lambda.data(), basis.rank(), c.w.data(), c.w.rows(),
      static_cast<int32_t>(c.w.cols()), out.pts.data()));
  return out;
}

// solvers.hpp:160-176 — σ² by the trace form (P row-constrained).
inline double update_sigma2(const PointSet& y, const Correspondence& p, const PointSet& x_t) {
  if (!p.row_constrained) throw ParameterError("update_sigma2 requires a row-constrained P");
  double out = 0.0;
  detail::l2check(fcpd_update_sigma2(detail::l2ctx(), y.pts.data(), y.count(), p.p.data(),
                                     p.p.rows(), p.p.cols(), x_t.pts.data(), x_t.count(),
                                     static_cast<int32_t>(x_t.dim()), 1, &out));
  return out;
}

// ------------------------------------------------------ pointset.hpp:31-148
struct NormalizationRecord {
  Vector center;
  double scale = 1.0;
  bool degenerate = false;

  PointSet apply(const PointSet& ps) const {
    PointSet out;
    out.pts.resize(ps.count(), ps.dim());
    for (Index j = 0; j < ps.dim(); ++j)
      for (Index i = 0; i < ps.count(); ++i) out.pts(i, j) = (ps.pts(i, j) - center(j)) / scale;
    return out;
  }
  PointSet invert(const PointSet& ps) const {
    PointSet out;
    out.pts.resize(ps.count(), ps.dim());
    for (Index j = 0; j < ps.dim(); ++j)
      for (Index i = 0; i < ps.count(); ++i) out.pts(i, j) = ps.pts(i, j) * scale + center(j);
    return out;
  }
};

// pointset.hpp:124-148 — joint centroid, max-abs scale, the same map on both.
inline std::tuple<PointSet, PointSet, NormalizationRecord> normalize_pair(const PointSet& x,
                                                                         const PointSet& y) {
  if (x.count() == 0 || y.count() == 0) throw ParameterError("normalize_pair: empty point set");
  if (x.dim() != y.dim()) throw DimensionError("normalize_pair: dimension mismatch");
  PointSet xo, yo;
  xo.pts.resize(x.count(), x.dim());
  yo.pts.resize(y.count(), y.dim());
  NormalizationRecord rec;
  rec.center.resize(x.dim());
  int32_t deg = 0;
  detail::l2check(fcpd_normalize_pair(detail::l2ctx(), x.pts.data(), x.count(),
                                      static_cast<int32_t>(x.dim()), y.pts.data(), y.count(),
                                      static_cast<int32_t>(y.dim()), xo.pts.data(),
                                      yo.pts.data(), rec.center.data(), &rec.scale, &deg));
  rec.degenerate = deg != 0;
  return {std::move(xo), std::move(yo), rec};
}

// registration.hpp:59-69 (host, O(M+N)).
inline double init_sigma2(const PointSet& x, const PointSet& y) {
  if (x.count() == 0 || y.count() == 0) throw ParameterError("init_sigma2: empty point set");
  if (x.dim() != y.dim()) throw DimensionError("init_sigma2: dimension mismatch");
  const double m = static_cast<double>(x.count()), n = static_cast<double>(y.count());
  double fx = 0, fy = 0, dot = 0;
  for (Index j = 0; j < x.dim(); ++j) {
    double sx = 0, sy = 0;
    for (Index i = 0; i < x.count(); ++i) {
      fx += x.pts(i, j) * x.pts(i, j);
      sx += x.pts(i, j);
    }
    for (Index i = 0; i < y.count(); ++i) {
      fy += y.pts(i, j) * y.pts(i, j);
      sy += y.pts(i, j);
    }
    dot += sx * sy;
  }
  const double v = (m * fy + n * fx - 2.0 * dot) / (static_cast<double>(x.dim()) * m * n);
  return v > 0.0 ? v : 0.0;
}

// ------------------------------------------- point files (pointset.hpp:45-119)
// Text point files: one point per line, coordinates separated by whitespace
// or commas, '#' starts a comment, blank lines ignored.  Same checks and
// messages as the reference: unreadable file → IoError, a token that is not
// a finite number → ParseError "path:line: malformed number 'tok'", a row
// of another width → DimensionError, no points → ParseError.
inline PointSet load_points(const std::string& path, Index expected_dim = -1) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open point file: " + path);
  std::vector<double> vals;
  Index dim = -1, rows = 0;
  std::string line;
  long lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    std::replace(line.begin(), line.end(), ',', ' ');
    std::istringstream ss(line);
    std::string tok;
    Index width = 0;
    while (ss >> tok) {
      if (tok[0] == '#') break;
      char* end = nullptr;
      errno = 0;
      const double v = std::strtod(tok.c_str(), &end);
      if (end != tok.c_str() + tok.size() || !std::isfinite(v) || tok.empty())
        throw ParseError(path + ":" + std::to_string(lineno) + ": malformed number '" + tok +
                         "'");
      vals.push_back(v);
      ++width;
    }
    if (width == 0) continue;  // blank or comment-only line
    if (dim < 0) dim = width;
    else if (width != dim)
      throw DimensionError(path + ":" + std::to_string(lineno) + ": expected " +
                           std::to_string(dim) + " columns, got " + std::to_string(width));
    ++rows;
  }
  if (rows == 0) throw ParseError(path + ": no points in file");
  if (expected_dim >= 0 && dim != expected_dim)
    throw DimensionError(path + ": expected dimension " + std::to_string(expected_dim) +
                         ", got " + std::to_string(dim));
  Matrix m(rows, dim);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < dim; ++j) m(i, j) = vals[static_cast<size_t>(i * dim + j)];
  return PointSet{std::move(m)};
}

// Full round-trip precision (max_digits10), one point per line.
inline void write_points(const PointSet& ps, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open for writing: " + path);
  out.precision(std::numeric_limits<double>::max_digits10);
  for (Index i = 0; i < ps.count(); ++i) {
    for (Index j = 0; j < ps.dim(); ++j) out << (j ? " " : "") << ps.pts(i, j);
    out << '\n';
  }
  if (!out) throw IoError("write failed: " + path);
}

// ------------------------------------------- run report (registration.hpp:178-204)
// key=value lines (15 significant digits): the configuration, diagnostics,
// timing breakdown and the σ² trace as sigma2[i]=….  The device run adds
// t_setup (Gram + eigendecomposition) after t_total.
inline void write_report(const std::string& path, const RegistrationConfig& cfg,
                         const RegistrationResult& res) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot write report: " + path);
  out.precision(15);
  const auto kv = [&](const char* k, auto v) { out << k << '=' << v << '\n'; };
  kv("variant", to_string(cfg.variant));
  kv("omega", cfg.omega);
  kv("beta", cfg.beta);
  kv("lambda", cfg.lambda_reg);
  kv("iterations", cfg.iterations);
  kv("rank_fraction", cfg.rank_fraction);
  kv("seed", cfg.seed);
  kv("normalize", cfg.normalize ? 1 : 0);
  kv("baseline_solver", res.diagnostics.baseline_solver);
  kv("sigma2_initial", res.sigma2_initial);
  kv("degenerate_rows", res.diagnostics.degenerate_rows);
  kv("sigma2_clamps", res.diagnostics.sigma2_clamps);
  kv("t_c", res.timing.t_c);
  kv("t_eig", res.timing.t_eig);
  kv("t_iter", res.timing.t_iter);
  kv("t_f", res.timing.t_f);
  kv("t_o", res.timing.t_o);
  kv("t_total", res.timing.t_total);
  kv("t_setup", res.timing.t_setup);
  for (size_t i = 0; i < res.sigma2_trace.size(); ++i)
    out << "sigma2[" << i << "]=" << res.sigma2_trace[i] << '\n';
  if (!out) throw IoError("report write failed: " + path);
}

// ------------------------------------------- benchmark harness (metrics.hpp)
// Ground truth: model row index → expected position (degradations.hpp:22).
using Truth = std::map<Index, std::vector<double>>;

struct DegradedPair {
  PointSet model;
  PointSet scene;
  Truth truth;
};

// RMS distance of the transformed model rows that have a ground truth
// (metrics.hpp:19-31).
inline double rmse(const PointSet& transformed, const Truth& truth) {
  if (truth.empty()) throw ParameterError("rmse: empty ground truth");
  double sum = 0.0;
  for (const auto& kv : truth) {
    const Index i = kv.first;
    if (i < 0 || i >= transformed.count()) throw ParameterError("rmse: truth index out of range");
    if (static_cast<Index>(kv.second.size()) != transformed.dim())
      throw DimensionError("rmse: truth dimension mismatch");
    for (Index j = 0; j < transformed.dim(); ++j) {
      const double e = transformed.pts(i, j) - kv.second[static_cast<size_t>(j)];
      sum += e * e;
    }
  }
  return std::sqrt(sum / static_cast<double>(truth.size()));
}

struct BenchRecord {
  Index m = 0, n = 0;
  SolverVariant variant = SolverVariant::fast;
  TimingBreakdown timing;
  double rmse = 0.0;
  int iterations = 0;
  bool failed = false;
};

// `size` rows drawn without replacement, kept in source order, deterministic
// per seed (metrics.hpp:43-58).
inline PointSet subsample(const PointSet& ps, Index size, unsigned long seed) {
  if (size < 1 || size > ps.count()) throw ParameterError("subsample: size out of range");
  std::vector<Index> idx(static_cast<size_t>(ps.count()));
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<Index>(i);
  std::mt19937_64 rng(seed);
  std::shuffle(idx.begin(), idx.end(), rng);
  idx.resize(static_cast<size_t>(size));
  std::sort(idx.begin(), idx.end());
  PointSet out;
  out.pts.resize(size, ps.dim());
  for (Index i = 0; i < size; ++i)
    for (Index j = 0; j < ps.dim(); ++j) out.pts(i, j) = ps.pts(idx[static_cast<size_t>(i)], j);
  return out;
}

// A mild random affine map (metrics.hpp:60-94): rotation ≤ 10° (about a
// random axis in 3-D), per-axis scale in [0.9, 1.1], shift in [−0.1, 0.1].
inline PointSet random_affine(const PointSet& ps, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  const Index d = ps.dim();
  const double max_angle = 10.0 * 3.14159265358979323846 / 180.0;
  double rot[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  if (d == 2) {
    const double a = unit(rng) * max_angle;
    rot[0][0] = std::cos(a), rot[0][1] = -std::sin(a);
    rot[1][0] = std::sin(a), rot[1][1] = std::cos(a);
  } else if (d == 3) {
    double ax[3] = {unit(rng), unit(rng), unit(rng)};
    double nrm = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    if (nrm < 1e-12) ax[0] = ax[1] = 0.0, ax[2] = 1.0, nrm = 1.0;
    for (double& c : ax) c /= nrm;
    const double a = unit(rng) * max_angle, sa = std::sin(a), ca = 1.0 - std::cos(a);
    const double k[3][3] = {{0, -ax[2], ax[1]}, {ax[2], 0, -ax[0]}, {-ax[1], ax[0], 0}};
    for (int i = 0; i < 3; ++i)  // Rodrigues: I + sin(a)·K + (1 − cos(a))·K²
      for (int j = 0; j < 3; ++j) {
        double k2 = 0.0;
        for (int l = 0; l < 3; ++l) k2 += k[i][l] * k[l][j];
        rot[i][j] = (i == j ? 1.0 : 0.0) + sa * k[i][j] + ca * k2;
      }
  }
  std::vector<double> scale(static_cast<size_t>(d)), shift(static_cast<size_t>(d));
  for (Index j = 0; j < d; ++j) {
    scale[static_cast<size_t>(j)] = 1.0 + 0.1 * unit(rng);
    shift[static_cast<size_t>(j)] = 0.1 * unit(rng);
  }
  PointSet out;
  out.pts.resize(ps.count(), d);
  for (Index i = 0; i < ps.count(); ++i)
    for (Index j = 0; j < d; ++j) {
      double v = 0.0;  // (p · Rᵀ)_j
      for (Index l = 0; l < d && l < 3; ++l) v += ps.pts(i, l) * rot[j][l];
      if (d > 3) v = ps.pts(i, j);
      out.pts(i, j) = v * scale[static_cast<size_t>(j)] + shift[static_cast<size_t>(j)];
    }
  return out;
}

// Scene = the subsample rescaled to [−1, 1] (joint normalisation with
// itself), model = its random-affine copy, truth row-to-row (metrics.hpp:96-106).
inline DegradedPair make_bench_pair(const PointSet& source, Index size, unsigned long seed) {
  const PointSet base = subsample(source, size, seed);
  const Index m = base.count(), d = base.dim();
  std::vector<double> ctr(static_cast<size_t>(d), 0.0);
  for (Index j = 0; j < d; ++j) {
    for (Index i = 0; i < m; ++i) ctr[static_cast<size_t>(j)] += 2.0 * base.pts(i, j);
    ctr[static_cast<size_t>(j)] /= static_cast<double>(2 * m);
  }
  double sc = 0.0;
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j)
      sc = std::max(sc, std::fabs(base.pts(i, j) - ctr[static_cast<size_t>(j)]));
  if (sc <= 0.0) sc = 1.0;
  DegradedPair pair;
  pair.scene.pts.resize(m, d);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j)
      pair.scene.pts(i, j) = (base.pts(i, j) - ctr[static_cast<size_t>(j)]) / sc;
  pair.model = random_affine(pair.scene, seed + 1);
  for (Index i = 0; i < m; ++i) {
    std::vector<double> row(static_cast<size_t>(d));
    for (Index j = 0; j < d; ++j) row[static_cast<size_t>(j)] = pair.scene.pts(i, j);
    pair.truth[i] = std::move(row);
  }
  return pair;
}

// One registration per (size, variant) cell, sequential, one discarded
// 1-iteration warm-up per size; a failing cell is recorded (rmse −1 in the
// CSV), not fatal (metrics.hpp:108-141).  On the device the cpd / cpd_lowrank
// variants are such failing cells.
inline std::vector<BenchRecord> run_benchmark(const PointSet& source,
                                              const std::vector<Index>& sizes,
                                              const std::vector<SolverVariant>& variants,
                                              const RegistrationConfig& cfg, unsigned long seed) {
  std::vector<BenchRecord> records;
  for (Index size : sizes) {
    const DegradedPair pair = make_bench_pair(source, size, seed + static_cast<unsigned long>(size));
    {
      RegistrationConfig warm = cfg;
      warm.iterations = 1;
      warm.variant = SolverVariant::fast;
      register_pointsets(pair.model, pair.scene, warm);
    }
    for (SolverVariant v : variants) {
      BenchRecord rec;
      rec.m = pair.model.count();
      rec.n = pair.scene.count();
      rec.variant = v;
      rec.iterations = cfg.iterations;
      try {
        RegistrationConfig run = cfg;
        run.variant = v;
        const RegistrationResult res = register_pointsets(pair.model, pair.scene, run);
        rec.timing = res.timing;
        rec.rmse = rmse(res.transformed, pair.truth);
      } catch (const Error&) {
        rec.failed = true;
      }
      records.push_back(rec);
    }
  }
  return records;
}

inline constexpr const char* kBenchCsvHeader =
    "M,N,variant,t_c,t_eig,t_iter,t_f,t_o,t_total,rmse,iterations";

// Durations with 6 decimals; t_f and t_total re-derived from the rounded
// parts so the timing identities hold exactly in the file (metrics.hpp:147-169).
inline void write_bench_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot write CSV: " + path);
  out << kBenchCsvHeader << '\n';
  const auto q = [](double v) { return std::round(v * 1e6) / 1e6; };
  char buf[512];
  for (const BenchRecord& r : records) {
    const double tc = q(r.timing.t_c), te = q(r.timing.t_eig), ti = q(r.timing.t_iter),
                 to = q(r.timing.t_o);
    std::snprintf(buf, sizeof buf, "%lld,%lld,%s,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.9g,%d\n",
                  static_cast<long long>(r.m), static_cast<long long>(r.n), to_string(r.variant),
                  tc, te, ti, te + ti, to, tc + te + ti + to, r.failed ? -1.0 : r.rmse,
                  r.iterations);
    out << buf;
  }
  if (!out) throw IoError("CSV write failed: " + path);
}

inline std::vector<BenchRecord> load_bench_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open CSV: " + path);
  std::string line;
  if (!std::getline(in, line) || line != kBenchCsvHeader)
    throw ParseError(path + ": missing or unexpected CSV header");
  std::vector<BenchRecord> records;
  long lineno = 1;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    std::vector<std::string> cells;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) cells.push_back(cell);
    if (!line.empty() && line.back() == ',') cells.push_back("");
    if (cells.size() != 11) throw ParseError(path + ":" + std::to_string(lineno) + ": bad CSV row");
    BenchRecord r;
    try {
      r.m = std::stoll(cells[0]);
      r.n = std::stoll(cells[1]);
      r.variant = variant_from_string(cells[2]);
      r.timing.t_c = std::stod(cells[3]);
      r.timing.t_eig = std::stod(cells[4]);
      r.timing.t_iter = std::stod(cells[5]);
      r.timing.t_f = std::stod(cells[6]);
      r.timing.t_o = std::stod(cells[7]);
      r.timing.t_total = std::stod(cells[8]);
      r.rmse = std::stod(cells[9]);
      r.iterations = std::stoi(cells[10]);
    } catch (const ParameterError&) {
      throw ParseError(path + ":" + std::to_string(lineno) + ": bad CSV value");
    } catch (const std::exception&) {
      throw ParseError(path + ":" + std::to_string(lineno) + ": bad CSV value");
    }
    r.failed = r.rmse < 0.0;
    records.push_back(r);
  }
  return records;
}

// Log-log chart of t_iter against M, one path per variant, as an SVG string
// (the reference's svg::bench_plot, svg.hpp:81-133): deterministic output,
// failed cells and non-positive values skipped, an empty chart shell when
// nothing is left.
inline std::string bench_plot(const std::vector<BenchRecord>& records) {
  constexpr double kW = 480, kH = 360, kLeft = 60, kRight = 20, kTop = 20, kBottom = 50;
  static const char* kColors[] = {"#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e",
                                  "#8c564b"};
  const auto num = [](double v) {
    char b[32];
    std::snprintf(b, sizeof b, "%.2f", v);
    return std::string(b);
  };
  std::map<std::string, std::vector<std::pair<double, double>>> series;
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (const BenchRecord& r : records) {
    if (r.failed || r.m <= 0 || !(r.timing.t_iter > 0.0)) continue;
    const double x = std::log10(static_cast<double>(r.m)), y = std::log10(r.timing.t_iter);
    series[to_string(r.variant)].emplace_back(x, y);
    x0 = std::min(x0, x), x1 = std::max(x1, x);
    y0 = std::min(y0, y), y1 = std::max(y1, y);
  }
  // data → pixel along one axis (a degenerate range maps to the middle)
  const auto axis = [](double v, double lo, double hi, double p0, double p1) {
    return hi > lo ? p0 + (v - lo) / (hi - lo) * (p1 - p0) : 0.5 * (p0 + p1);
  };
  std::string out = "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" + num(kW) +
                    "\" height=\"" + num(kH) + "\">\n";
  out += "<rect x=\"" + num(kLeft) + "\" y=\"" + num(kTop) + "\" width=\"" +
         num(kW - kLeft - kRight) + "\" height=\"" + num(kH - kTop - kBottom) +
         "\" fill=\"none\" stroke=\"#000000\"/>\n";
  out += "<text x=\"" + num(kW / 2) + "\" y=\"" + num(kH - 10) +
         "\" text-anchor=\"middle\" font-size=\"14\">M (log scale)</text>\n";
  out += "<text x=\"15\" y=\"" + num(kH / 2) +
         "\" text-anchor=\"middle\" font-size=\"14\" transform=\"rotate(-90 15 " + num(kH / 2) +
         ")\">t_iter seconds (log scale)</text>\n";
  int k = 0;
  for (auto& [name, pts] : series) {
    std::sort(pts.begin(), pts.end());
    std::string d;
    for (size_t i = 0; i < pts.size(); ++i)
      d += (i ? " L " : "M ") + num(axis(pts[i].first, x0, x1, kLeft, kW - kRight)) + " " +
           num(axis(pts[i].second, y0, y1, kH - kBottom, kTop));
    const char* col = kColors[k % 6];
    ++k;
    out += "<path d=\"" + d + "\" fill=\"none\" stroke=\"" + col + "\" stroke-width=\"2\"/>\n";
    out += "<text x=\"" + num(kW - kRight - 5) + "\" y=\"" + num(kTop + 15.0 * k) +
           "\" text-anchor=\"end\" font-size=\"12\" fill=\"" + col + "\">" + name + "</text>\n";
  }
  out += "</svg>\n";
  return out;
}

inline void write_text_file(const std::string& content, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot write file: " + path);
  out << content;
  if (!out) throw IoError("write failed: " + path);
}

}  // namespace fastcpd
