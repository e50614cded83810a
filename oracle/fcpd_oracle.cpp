// fcpd_oracle.cpp — CPU fp64 restatement of the reference Fast-CPD hot path.
//
// TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it.  It is never on the product path.
//
// The reference (/root/reference/proj/include/fastcpd/*.hpp) is header-only
// C++/Eigen and cannot be compiled in this image (Eigen3 and vendor/ absent,
// see DESIGN.md §Oracle).  Every function below restates one reference
// function in plain fp64 C++ with the same operation order where it matters
// (shift, clamp, floor, throw conditions).  Matrices are column-major like
// Eigen::MatrixXd, so a PointSet of M points in D dims is SoA: x[d*M + m].
//
// Parity pin: the known-answer tests of proj/tests/*.cpp are ported into
// tests/test_oracle_kat.py, and tests/golden/make_golden.py (an independent
// numpy restatement) cross-checks full registrations.
//
// Eigensolver: LAPACK dsyevd from the scipy-bundled OpenBLAS (dlopen'ed), in
// place of Eigen::SelfAdjointEigenSolver (kernel.hpp:54).  Different
// algorithm, same eigenpairs up to rounding for resolved eigenvalues.

#include <dlfcn.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

// Error codes shared with include/fcpd_capi.h.
enum : int {
  kOk = 0,
  kParameter = 1,
  kDimension = 2,
  kNumeric = 3,
  kIo = 4,
  kParse = 5,
};

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

constexpr double kSigma2Floor = 1e-10;  // correspondence.hpp:12

// ---------------------------------------------------------------- LAPACK ---
using dsyevd_t = void (*)(const char*, const char*, const int*, double*,
                          const int*, double*, double*, const int*, int*,
                          const int*, int*);
using dposv_t = void (*)(const char*, const int*, const int*, double*,
                         const int*, double*, const int*, int*);
using setthreads_t = void (*)(int);

struct Lapack {
  dsyevd_t dsyevd = nullptr;
  dposv_t dposv = nullptr;
  setthreads_t set_threads = nullptr;
  std::string err;
};

Lapack& lapack() {
  static Lapack L = [] {
    Lapack l;
    const char* env = std::getenv("FCPD_ORACLE_LAPACK");
    const char* cands[] = {
        env,
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/scipy.libs/"
        "libscipy_openblas-5f890258.so",
    };
    void* h = nullptr;
    for (const char* c : cands) {
      if (!c) continue;
      h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      l.err = "oracle: cannot dlopen scipy OpenBLAS (set FCPD_ORACLE_LAPACK)";
      return l;
    }
    l.dsyevd = reinterpret_cast<dsyevd_t>(dlsym(h, "scipy_dsyevd_"));
    l.dposv = reinterpret_cast<dposv_t>(dlsym(h, "scipy_dposv_"));
    l.set_threads =
        reinterpret_cast<setthreads_t>(dlsym(h, "scipy_openblas_set_num_threads"));
    if (!l.dsyevd) l.err = "oracle: scipy_dsyevd_ not found";
    return l;
  }();
  return L;
}

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// Column-major helpers (Eigen::MatrixXd layout).
inline double& at(double* a, int64_t ld, int64_t i, int64_t j) {
  return a[j * ld + i];
}
inline double at(const double* a, int64_t ld, int64_t i, int64_t j) {
  return a[j * ld + i];
}

// out (M×d, column-major) = (x0 or 0) + U·Z, U M×k column-major, Z k×d
// column-major with leading dimension ldz (default k).  Each thread owns a
// block of rows and streams the columns of U through it: the same sums as
// the naive per-row loop (Σ_i in increasing i), but cache-friendly.
void basis_times(const double* u, int64_t m, int64_t k, const double* z, int d,
                 const double* x0, double* out, int64_t ldz = 0) {
  constexpr int64_t kRows = 512;
  if (ldz == 0) ldz = k;
#pragma omp parallel for schedule(static)
  for (int64_t r0 = 0; r0 < m; r0 += kRows) {
    const int64_t r1 = std::min(m, r0 + kRows);
    double acc[3][kRows];
    for (int j = 0; j < d; ++j)
      for (int64_t r = r0; r < r1; ++r) acc[j][r - r0] = 0.0;
    for (int64_t i = 0; i < k; ++i) {
      const double* ui = u + i * m;
      for (int j = 0; j < d; ++j) {
        const double zi = z[j * ldz + i];
        for (int64_t r = r0; r < r1; ++r) acc[j][r - r0] += ui[r] * zi;
      }
    }
    for (int j = 0; j < d; ++j)
      for (int64_t r = r0; r < r1; ++r)
        out[j * m + r] = (x0 ? x0[j * m + r] : 0.0) + acc[j][r - r0];
  }
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void orc_set_threads(int n) {
  if (n < 1) n = 1;
  omp_set_num_threads(n);
  if (lapack().set_threads) lapack().set_threads(n);
}

int orc_get_threads() { return omp_get_max_threads(); }

// pointset.hpp:124-148 normalize_pair.  Outputs xo (M×D), yo (N×D), center (D).
int orc_normalize_pair(const double* x, int64_t m, const double* y, int64_t n,
                       int d, double* xo, double* yo, double* center,
                       double* scale, int* degenerate) {
  if (m == 0 || n == 0) return fail(kParameter, "normalize_pair: empty point set");
  const double total = static_cast<double>(m + n);
  for (int j = 0; j < d; ++j) {
    double sx = 0.0, sy = 0.0;  // colwise().sum() of each set, then added
    for (int64_t i = 0; i < m; ++i) sx += at(x, m, i, j);
    for (int64_t i = 0; i < n; ++i) sy += at(y, n, i, j);
    center[j] = (sx + sy) / total;
  }
  double s = 0.0;
  for (int j = 0; j < d; ++j) {
    for (int64_t i = 0; i < m; ++i) s = std::max(s, std::fabs(at(x, m, i, j) - center[j]));
    for (int64_t i = 0; i < n; ++i) s = std::max(s, std::fabs(at(y, n, i, j) - center[j]));
  }
  *degenerate = 0;
  if (s <= 0.0) {
    s = 1.0;
    *degenerate = 1;
  }
  *scale = s;
  for (int j = 0; j < d; ++j) {
    for (int64_t i = 0; i < m; ++i) at(xo, m, i, j) = (at(x, m, i, j) - center[j]) / s;
    for (int64_t i = 0; i < n; ++i) at(yo, n, i, j) = (at(y, n, i, j) - center[j]) / s;
  }
  return kOk;
}

// registration.hpp:59-69 init_sigma2.
int orc_init_sigma2(const double* x, int64_t m, const double* y, int64_t n,
                    int d, double* out) {
  if (m == 0 || n == 0) return fail(kParameter, "init_sigma2: empty point set");
  double fx = 0.0, fy = 0.0, dot = 0.0;
  for (int j = 0; j < d; ++j) {
    double sx = 0.0, sy = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double v = at(x, m, i, j);
      fx += v * v;
      sx += v;
    }
    for (int64_t i = 0; i < n; ++i) {
      const double v = at(y, n, i, j);
      fy += v * v;
      sy += v;
    }
    dot += sx * sy;
  }
  const double md = static_cast<double>(m), nd = static_cast<double>(n);
  const double sum = md * fy + nd * fx - 2.0 * dot;
  *out = std::max(sum / (static_cast<double>(d) * md * nd), 0.0);
  return kOk;
}

// kernel.hpp:31-47 build_gram.  phi is M×M column-major.
int orc_build_gram(const double* x, int64_t m, int d, double beta, double* phi) {
  if (beta <= 0.0) return fail(kParameter, "build_gram: beta must be positive");
  const double inv = 1.0 / (2.0 * beta * beta);
  std::vector<double> sq(m, 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int j = 0; j < d; ++j) sq[i] += at(x, m, i, j) * at(x, m, i, j);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < m; ++c) {
    for (int64_t r = 0; r < m; ++r) {
      double xy = 0.0;
      for (int j = 0; j < d; ++j) xy += at(x, m, r, j) * at(x, m, c, j);
      const double d2 = sq[r] + sq[c] - 2.0 * xy;
      at(phi, m, r, c) = std::exp(-std::max(d2, 0.0) * inv);
    }
  }
  // symmetrise exactly and pin the diagonal (kernel.hpp:44-45)
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t c = 0; c < m; ++c) {
    for (int64_t r = c + 1; r < m; ++r) {
      const double s = (at(phi, m, r, c) + at(phi, m, c, r)) * 0.5;
      at(phi, m, r, c) = s;
      at(phi, m, c, r) = s;
    }
    at(phi, m, c, c) = 1.0;
  }
  return kOk;
}

// kernel.hpp:49-72 eigendecompose: top-`rank` eigenpairs, descending, with
// the 1e-12·λmax clamp.  u is M×rank column-major.  lambda_raw (optional)
// receives the unclamped values.
int orc_eigendecompose(const double* phi, int64_t m, int64_t rank, double* u,
                       double* lambda, double* lambda_raw) {
  if (rank < 1 || rank > m) return fail(kParameter, "eigendecompose: rank out of [1, M]");
  Lapack& L = lapack();
  if (!L.dsyevd) return fail(kNumeric, L.err);
  if (m > 46340) return fail(kParameter, "eigendecompose: M too large for the dense oracle");
  std::vector<double> a(phi, phi + m * m);
  std::vector<double> w(m);
  const int n = static_cast<int>(m);
  int info = 0, lwork = -1, liwork = -1, iwq = 0;
  double wq = 0.0;
  L.dsyevd("V", "L", &n, a.data(), &n, w.data(), &wq, &lwork, &iwq, &liwork, &info);
  lwork = static_cast<int>(wq) + 1;
  liwork = iwq;
  std::vector<double> work(lwork);
  std::vector<int> iwork(liwork);
  L.dsyevd("V", "L", &n, a.data(), &n, w.data(), work.data(), &lwork,
           iwork.data(), &liwork, &info);
  if (info != 0)
    return fail(kNumeric, "eigendecompose: symmetric eigensolver did not converge (info=" +
                              std::to_string(info) + ")");
  // ascending → take the top `rank` reversed (kernel.hpp:59-66)
  for (int64_t i = 0; i < rank; ++i) {
    const int64_t src = m - 1 - i;
    std::memcpy(u + i * m, a.data() + src * m, sizeof(double) * m);
    lambda[i] = w[src];
    if (lambda_raw) lambda_raw[i] = w[src];
  }
  const double floor = 1e-12 * std::max(lambda[0], 0.0);  // kernel.hpp:68-70
  for (int64_t i = 0; i < rank; ++i)
    if (lambda[i] < floor) lambda[i] = 0.0;
  return kOk;
}

// correspondence.hpp:35-79 posterior.  p is M×N column-major.
int orc_posterior(const double* xt, int64_t m, const double* y, int64_t n,
                  int d, double omega, double sigma2, double* p, int* clamped) {
  if (omega < 0.0 || omega >= 1.0)
    return fail(kParameter, "posterior: omega must lie in [0, 1)");
  *clamped = 0;
  if (sigma2 < kSigma2Floor) {
    sigma2 = kSigma2Floor;
    *clamped = 1;
  }
  const double inv = 1.0 / (2.0 * sigma2);
  std::vector<double> sx(m, 0.0), sy(n, 0.0);
  for (int j = 0; j < d; ++j) {
    for (int64_t i = 0; i < m; ++i) sx[i] += at(xt, m, i, j) * at(xt, m, i, j);
    for (int64_t i = 0; i < n; ++i) sy[i] += at(y, n, i, j) * at(y, n, i, j);
  }
  const bool has_outlier = omega > 0.0;
  const double log_c =
      has_outlier ? 0.5 * d * std::log(2.0 * M_PI * sigma2) +
                        std::log(omega / (1.0 - omega)) +
                        std::log(static_cast<double>(m) / static_cast<double>(n))
                  : 0.0;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double* col = p + c * m;
    // expo = -max(sx + sy - 2 x·y, 0) * inv   (correspondence.hpp:56-59)
    double shift = -INFINITY;
    for (int64_t r = 0; r < m; ++r) {
      double xy = 0.0;
      for (int j = 0; j < d; ++j) xy += at(xt, m, r, j) * at(y, n, c, j);
      const double e = -std::max(sx[r] + sy[c] - 2.0 * xy, 0.0) * inv;
      col[r] = e;
      shift = std::max(shift, e);
    }
    if (has_outlier && log_c > shift) shift = log_c;
    double denom = 0.0;
    for (int64_t r = 0; r < m; ++r) {
      col[r] = std::exp(col[r] - shift);
      denom += col[r];
    }
    if (has_outlier) denom += std::exp(log_c - shift);
    for (int64_t r = 0; r < m; ++r) col[r] /= denom;
  }
  return kOk;
}

// correspondence.hpp:83-98 enforce_row_constraint, in place on p (M×N).
// degenerate (optional, length M) receives 1 for rows replaced by uniform.
int orc_enforce_row_constraint(double* p, int64_t m, int64_t n,
                               int64_t* degenerate_rows, int64_t* n_degenerate) {
  std::vector<double> s(m, 0.0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) s[r] += p[c * m + r];
  int64_t nd = 0;
  for (int64_t r = 0; r < m; ++r) {
    if (s[r] < 1e-300) {
      for (int64_t c = 0; c < n; ++c) p[c * m + r] = 1.0 / static_cast<double>(n);
      if (degenerate_rows) degenerate_rows[nd] = r;
      ++nd;
    } else {
      for (int64_t c = 0; c < n; ++c) p[c * m + r] /= s[r];
    }
  }
  *n_degenerate = nd;
  return kOk;
}

// correspondence.hpp:101-105 estimated_targets: out = P·Y (M×D).
int orc_estimated_targets(const double* p, int64_t m, int64_t n, const double* y,
                          int64_t ny, int d, double* out) {
  if (n != ny) return fail(kParameter, "estimated_targets: shape mismatch");
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int64_t c = 0; c < n; ++c) acc += p[c * m + r] * y[j * n + c];
      out[j * m + r] = acc;
    }
  }
  return kOk;
}

// solvers.hpp:61-73 solve_fast_lowrank: W = U diag(1/(λ+λ_reg σ²)) Uᵀ R.
int orc_solve_fast_lowrank(const double* u, const double* lambda, int64_t m,
                           int64_t k, double lambda_reg, double sigma2,
                           const double* residual, int64_t rm, int d, double* w) {
  if (rm != m) return fail(kParameter, "solve_fast: residual rows must match basis points");
  const double shift = lambda_reg * sigma2;
  double mn = INFINITY;
  for (int64_t i = 0; i < k; ++i) mn = std::min(mn, lambda[i] + shift);
  if (mn <= 0.0) return fail(kNumeric, "solve_fast: lambda_i + lambda*sigma2 not positive");
  std::vector<double> z(k * d, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) {
    const double* ui = u + i * m;
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int64_t r = 0; r < m; ++r) acc += ui[r] * residual[j * m + r];
      z[j * k + i] = acc / (lambda[i] + shift);
    }
  }
  basis_times(u, m, k, z.data(), d, nullptr, w);
  return kOk;
}

// solvers.hpp:138-144 apply_transform: out = X + Φ W.
int orc_apply_transform(const double* x, int64_t m, int d, const double* phi,
                        const double* w, double* out) {
  // out = X + Φ W: Φ column-major, streamed by columns (column c scaled by W_c)
  basis_times(phi, m, m, w, d, x, out, m);
  return kOk;
}

// solvers.hpp:147-155 apply_transform_lowrank: out = X + U Λ Uᵀ W.
int orc_apply_transform_lowrank(const double* x, int64_t m, int d, const double* u,
                                const double* lambda, int64_t k, const double* w,
                                double* out) {
  std::vector<double> t(k * d, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i)
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int64_t r = 0; r < m; ++r) acc += u[i * m + r] * w[j * m + r];
      t[j * k + i] = lambda[i] * acc;
    }
  basis_times(u, m, k, t.data(), d, x, out);
  return kOk;
}

// solvers.hpp:160-176 update_sigma2 (trace form).  p must be row-constrained.
int orc_update_sigma2(const double* y, int64_t n, const double* p, int64_t m,
                      const double* xt, int d, int row_constrained, double* out) {
  if (!row_constrained)
    return fail(kParameter, "update_sigma2 requires a row-constrained P");
  std::vector<double> pt1(n, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double s = 0.0;
    for (int64_t r = 0; r < m; ++r) s += p[c * m + r];
    pt1[c] = s;
  }
  double term1 = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    double sq = 0.0;
    for (int j = 0; j < d; ++j) sq += y[j * n + c] * y[j * n + c];
    term1 += sq * pt1[c];
  }
  std::vector<double> ytilde(m * d);
  orc_estimated_targets(p, m, n, y, n, d, ytilde.data());
  double term2 = 0.0, term3 = 0.0;
  for (int64_t i = 0; i < m * d; ++i) {
    term2 += ytilde[i] * xt[i];
    term3 += xt[i] * xt[i];
  }
  const double val = (term1 - 2.0 * term2 + term3) /
                     (static_cast<double>(d) * static_cast<double>(m));
  if (val < -1e-8)
    return fail(kNumeric, "update_sigma2: negative variance " + std::to_string(val));
  *out = std::max(val, kSigma2Floor);
  return kOk;
}

// solvers.hpp:85-104 solve_cpd_baseline (dense SPD solve; LDLT in the
// reference, Cholesky dposv here — same solution for the SPD system).
int orc_solve_cpd_baseline(const double* phi, int64_t m, const double* p, int64_t n,
                           double lambda_reg, double sigma2, const double* y,
                           const double* x, int d, double* w) {
  Lapack& L = lapack();
  if (!L.dposv) return fail(kNumeric, "oracle: dposv unavailable");
  std::vector<double> p1(m, 0.0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) p1[r] += p[c * m + r];
  std::vector<double> a(phi, phi + m * m);
  for (int64_t r = 0; r < m; ++r) {
    p1[r] = std::max(p1[r], 1e-10);
    a[r * m + r] += lambda_reg * sigma2 / p1[r];
  }
  std::vector<double> py(m * d);
  orc_estimated_targets(p, m, n, y, n, d, py.data());
  for (int j = 0; j < d; ++j)
    for (int64_t r = 0; r < m; ++r) w[j * m + r] = py[j * m + r] / p1[r] - x[j * m + r];
  const int nn = static_cast<int>(m), nrhs = d;
  int info = 0;
  L.dposv("L", &nn, &nrhs, a.data(), &nn, w, &nn, &info);
  if (info != 0) return fail(kNumeric, "solve_cpd_baseline: factorization failed");
  return kOk;
}

// ---------------------------------------------------------------------------
// Streaming (non-materialising) E-step: the exact algebra the device path
// uses, in fp64.  Outputs per model row m:
//   ptilde_y (M×D) = (P̃Y)_m, p1 (M) = raw row sum Σ_n P_mn,
//   var (M) = Σ_n P̃_mn ‖y_n − x̃_m‖², degenerate (M) flags; and per scene
//   column pt1 (N) = Σ_m P_mn (raw column mass, ≤ 1).
// Follows correspondence.hpp:35-98 + :101-105 semantics without forming P.
int orc_estep_stream(const double* xt, int64_t m, const double* y, int64_t n,
                     int d, double omega, double sigma2, double* ptilde_y,
                     double* p1, double* var, int32_t* degenerate, double* pt1,
                     int* clamped) {
  if (omega < 0.0 || omega >= 1.0)
    return fail(kParameter, "posterior: omega must lie in [0, 1)");
  *clamped = 0;
  if (sigma2 < kSigma2Floor) {
    sigma2 = kSigma2Floor;
    *clamped = 1;
  }
  const double inv = 1.0 / (2.0 * sigma2);
  const bool has_outlier = omega > 0.0;
  const double log_c =
      has_outlier ? 0.5 * d * std::log(2.0 * M_PI * sigma2) +
                        std::log(omega / (1.0 - omega)) +
                        std::log(static_cast<double>(m) / static_cast<double>(n))
                  : 0.0;
  auto d2 = [&](int64_t r, int64_t c) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      const double t = at(y, n, c, j) - at(xt, m, r, j);
      s += t * t;
    }
    return s;
  };
  // pass 1: column log-normaliser b_n = -(shift + log(denominator)).  Each
  // logit is formed once into a per-thread buffer; exp(a) for a < −746 is
  // exactly +0 in IEEE fp64 (the smallest subnormal is e^−744.44), so those
  // terms are skipped without changing a single bit of the sums.
  constexpr double kExpZero = -746.0;
  std::vector<double> b(n);
#pragma omp parallel
  {
    std::vector<double> e(m);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
      double mx = -INFINITY;
      for (int64_t r = 0; r < m; ++r) {
        e[r] = -d2(r, c) * inv;
        mx = std::max(mx, e[r]);
      }
      if (has_outlier && log_c > mx) mx = log_c;
      double sm = 0.0;
      for (int64_t r = 0; r < m; ++r) {
        const double a = e[r] - mx;
        if (a >= kExpZero) sm += std::exp(a);
      }
      const double s = sm + (has_outlier ? std::exp(log_c - mx) : 0.0);
      b[c] = -(mx + std::log(s));
      if (pt1) pt1[c] = sm / s;
    }
  }
  // column sums of y for the uniform fallback
  std::vector<double> ymean(d, 0.0);
  double ysq = 0.0;
  for (int j = 0; j < d; ++j) {
    for (int64_t c = 0; c < n; ++c) {
      ymean[j] += at(y, n, c, j);
      ysq += at(y, n, c, j) * at(y, n, c, j);
    }
    ymean[j] /= static_cast<double>(n);
  }
  ysq /= static_cast<double>(n);
  // pass 2: per row, max-shifted accumulation of w = exp(L - rowmax)
#pragma omp parallel
  {
    std::vector<double> lg(n);
#pragma omp for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    double mx = -INFINITY;
    for (int64_t c = 0; c < n; ++c) {
      lg[c] = -d2(r, c) * inv + b[c];
      mx = std::max(mx, lg[c]);
    }
    double s0 = 0.0, sv = 0.0;
    double sd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t c = 0; c < n; ++c) {
      const double a = lg[c] - mx;
      if (a < kExpZero) continue;  // w = +0 exactly
      const double dd = d2(r, c);
      const double wgt = std::exp(-dd * inv + b[c] - mx);
      s0 += wgt;
      sv += wgt * dd;
      for (int j = 0; j < d; ++j) sd[j] += wgt * (at(y, n, c, j) - at(xt, m, r, j));
    }
    const double logp1 = mx + std::log(s0);
    p1[r] = std::exp(logp1);
    if (logp1 < std::log(1e-300)) {  // row sum < 1e-300 → uniform row
      degenerate[r] = 1;
      double xsq = 0.0, xy = 0.0;
      for (int j = 0; j < d; ++j) {
        ptilde_y[j * m + r] = ymean[j];
        xsq += at(xt, m, r, j) * at(xt, m, r, j);
        xy += at(xt, m, r, j) * ymean[j];
      }
      var[r] = ysq - 2.0 * xy + xsq;
    } else {
      degenerate[r] = 0;
      for (int j = 0; j < d; ++j) ptilde_y[j * m + r] = at(xt, m, r, j) + sd[j] / s0;
      var[r] = sv / s0;
    }
  }
  }
  return kOk;
}

// ---------------------------------------------------------------------------
// registration.hpp:79-175 register_pointsets, fast / fast_lowrank variants,
// dense and faithful: P materialised, Φ materialised, full eigensolve.
//
// variant: 2 = fast, 3 = fast_lowrank (solvers.hpp:18 enum order).
// If basis_u/basis_lambda are non-null they replace the eigendecomposition
// (the paper's precomputed-basis protocol; used for bounded CPU samples).
// Outputs: out_x (M×D, original units), out_w (M×D), sigma2_trace
// (capacity `iterations`), iters_run, sigma2_initial, timing[6] =
// {t_c,t_eig,t_iter,t_f,t_o,t_total,t_loop}, diag[2] = {degenerate_rows, clamps}.
int orc_register(const double* x_in, int64_t m, const double* y_in, int64_t n,
                 int d, double omega, double beta, double lambda_reg,
                 int iterations, int variant, double rank_fraction, int normalize,
                 int early_stop, const double* basis_u, const double* basis_lambda,
                 int64_t basis_rank, double* out_x, double* out_w,
                 double* sigma2_trace, int* iters_run, double* sigma2_initial,
                 double* timing, int64_t* diag) {
  if (m == 0 || n == 0) return fail(kParameter, "register: empty point set");
  if (iterations < 0) return fail(kParameter, "register: negative iterations");
  if (variant != 2 && variant != 3)
    return fail(kParameter, "oracle register: only fast / fast_lowrank are restated");
  const auto t_start = Clock::now();
  double t_c = 0.0, t_eig = 0.0, t_iter = 0.0;

  std::vector<double> x(m * d), y(n * d), center(d, 0.0);
  double scale = 1.0;
  int degen = 0;
  if (normalize) {
    int rc = orc_normalize_pair(x_in, m, y_in, n, d, x.data(), y.data(),
                                center.data(), &scale, &degen);
    if (rc) return rc;
  } else {
    std::memcpy(x.data(), x_in, sizeof(double) * m * d);
    std::memcpy(y.data(), y_in, sizeof(double) * n * d);
  }
  const bool lowrank = variant == 3;
  int64_t rank = m;
  if (lowrank) {
    if (rank_fraction <= 0.0 || rank_fraction > 1.0)
      return fail(kParameter, "rank_fraction must lie in (0, 1]");
    rank = std::llround(rank_fraction * static_cast<double>(m));  // solvers.hpp:46-54
    rank = std::max<int64_t>(1, std::min<int64_t>(rank, m));
  }
  std::vector<double> phi;
  const bool need_phi = !lowrank || !basis_u;
  if (need_phi) {
    phi.resize(m * m);
    int rc = orc_build_gram(x.data(), m, d, beta, phi.data());
    if (rc) return rc;
  } else if (beta <= 0.0) {
    return fail(kParameter, "build_gram: beta must be positive");
  }
  std::vector<double> u, lam;
  if (basis_u) {
    if (basis_rank != rank) return fail(kParameter, "oracle register: basis rank mismatch");
    u.assign(basis_u, basis_u + m * rank);
    lam.assign(basis_lambda, basis_lambda + rank);
  } else {
    const auto t0 = Clock::now();
    u.resize(m * rank);
    lam.resize(rank);
    int rc = orc_eigendecompose(phi.data(), m, rank, u.data(), lam.data(), nullptr);
    if (rc) return rc;
    t_eig = since(t0);
  }
  double sigma2 = 0.0;
  orc_init_sigma2(x.data(), m, y.data(), n, d, &sigma2);
  *sigma2_initial = sigma2;

  std::vector<double> xt = x, w(m * d, 0.0), p(m * n), resid(m * d), wn(m * d),
                      xn(m * d);
  int64_t deg_total = 0, clamps = 0;
  int it = 0;
  const auto t_loop0 = Clock::now();
  for (; it < iterations; ++it) {
    const auto tc0 = Clock::now();
    int clamped = 0;
    int rc = orc_posterior(xt.data(), m, y.data(), n, d, omega, sigma2, p.data(), &clamped);
    if (rc) return fail(kNumeric, "register: iteration " + std::to_string(it) + ": " + g_err);
    if (clamped) ++clamps;
    int64_t nd = 0;
    orc_enforce_row_constraint(p.data(), m, n, nullptr, &nd);
    deg_total += nd;
    t_c += since(tc0);

    const auto ti0 = Clock::now();
    orc_estimated_targets(p.data(), m, n, y.data(), n, d, resid.data());
    for (int64_t i = 0; i < m * d; ++i) resid[i] -= x[i];
    rc = orc_solve_fast_lowrank(u.data(), lam.data(), m, rank, lambda_reg, sigma2,
                                resid.data(), m, d, wn.data());
    if (rc) return fail(kNumeric, "register: iteration " + std::to_string(it) + ": " + g_err);
    t_iter += since(ti0);

    if (lowrank)
      orc_apply_transform_lowrank(x.data(), m, d, u.data(), lam.data(), rank, wn.data(),
                                  xn.data());
    else
      orc_apply_transform(x.data(), m, d, phi.data(), wn.data(), xn.data());
    double next = 0.0;
    rc = orc_update_sigma2(y.data(), n, p.data(), m, xn.data(), d, 1, &next);
    if (rc) return fail(kNumeric, "register: iteration " + std::to_string(it) + ": " + g_err);
    if (next <= kSigma2Floor) ++clamps;
    xt.swap(xn);
    w.swap(wn);
    sigma2_trace[it] = next;
    const double delta = std::fabs(next - sigma2);
    sigma2 = next;
    if (early_stop && delta < 1e-10) {
      ++it;
      break;
    }
  }
  *iters_run = it;
  const double t_loop = since(t_loop0);
  for (int j = 0; j < d; ++j)
    for (int64_t r = 0; r < m; ++r)
      out_x[j * m + r] = normalize ? xt[j * m + r] * scale + center[j] : xt[j * m + r];
  std::memcpy(out_w, w.data(), sizeof(double) * m * d);
  const double t_f = t_eig + t_iter;
  const double measured = since(t_start);
  const double t_o = std::max(measured - t_c - t_f, 0.0);
  timing[0] = t_c;
  timing[1] = t_eig;
  timing[2] = t_iter;
  timing[3] = t_f;
  timing[4] = t_o;
  timing[5] = t_c + t_f + t_o;
  timing[6] = t_loop;  // EM loop only (bench's per-iteration CPU rate)
  diag[0] = deg_total;
  diag[1] = clamps;
  return kOk;
}

// ---------------------------------------------------------------------------
// Test fixtures restated from proj/tests/test_util.hpp:13-52 (std::mt19937_64
// with libstdc++'s distributions, so the inputs equal the reference tests').
// Outputs are column-major like Eigen.
// kernel.hpp:92-110 save_spectral_cache: "FCPD", u32 1, u64 M, u64 K,
// f64 beta, U row-major, λ.  u is column-major M×K here (Eigen layout).
int orc_save_spectral_cache(const char* path, const double* u, const double* lambda, int64_t m,
                            int64_t k, double beta) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(kIo, std::string("cannot open spectral cache for writing: ") + path);
  const uint32_t ver = 1;
  const uint64_t mm = m, kk = k;
  bool ok = std::fwrite("FCPD", 1, 4, f) == 4 && std::fwrite(&ver, 4, 1, f) == 1 &&
            std::fwrite(&mm, 8, 1, f) == 1 && std::fwrite(&kk, 8, 1, f) == 1 &&
            std::fwrite(&beta, 8, 1, f) == 1;
  std::vector<double> row(k);
  for (int64_t i = 0; ok && i < m; ++i) {
    for (int64_t j = 0; j < k; ++j) row[j] = u[j * m + i];
    ok = std::fwrite(row.data(), 8, k, f) == static_cast<size_t>(k);
  }
  ok = ok && std::fwrite(lambda, 8, k, f) == static_cast<size_t>(k);
  ok = (std::fclose(f) == 0) && ok;
  return ok ? kOk : fail(kIo, std::string("spectral cache write failed: ") + path);
}

// kernel.hpp:112-144 load_spectral_cache.  Call with u == nullptr to read
// the header only (m, k, beta).
int orc_load_spectral_cache(const char* path, int64_t* m, int64_t* k, double* beta, double* u,
                            double* lambda) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(kIo, std::string("cannot open spectral cache: ") + path);
  char magic[4];
  uint32_t ver = 0;
  uint64_t mm = 0, kk = 0;
  double b = 0.0;
  const bool hdr = std::fread(magic, 1, 4, f) == 4 && std::fread(&ver, 4, 1, f) == 1 &&
                   std::fread(&mm, 8, 1, f) == 1 && std::fread(&kk, 8, 1, f) == 1 &&
                   std::fread(&b, 8, 1, f) == 1;
  if (!hdr || std::memcmp(magic, "FCPD", 4) != 0) {
    std::fclose(f);
    return fail(kParse, std::string("not a spectral cache file: ") + path);
  }
  if (ver != 1) {
    std::fclose(f);
    return fail(kParse, std::string("unsupported spectral cache version in ") + path);
  }
  *m = static_cast<int64_t>(mm);
  *k = static_cast<int64_t>(kk);
  *beta = b;
  if (!u) {
    std::fclose(f);
    return kOk;
  }
  std::vector<double> row(kk);
  bool ok = true;
  for (uint64_t i = 0; ok && i < mm; ++i) {
    ok = std::fread(row.data(), 8, kk, f) == kk;
    for (uint64_t j = 0; j < kk; ++j) u[j * mm + i] = row[j];
  }
  ok = ok && std::fread(lambda, 8, kk, f) == kk;
  std::fclose(f);
  return ok ? kOk : fail(kParse, std::string("truncated spectral cache: ") + path);
}

// register_pointsets (registration.hpp:79-175) for a GIVEN basis with the
// streaming E-step (orc_estep_stream: no M×N matrix) — the oracle for
// configs whose dense P (20–320 GB) does not fit.  Transform: X + U
// diag(λ_num) Uᵀ W (λ_num = raw λ for full rank, clamped for low rank);
// σ² by the per-row form Σ_m [V_m − 2δ·Δ̄ + ‖δ‖²]/(DM), algebraically the
// trace form of solvers.hpp:166-172 (row sums of P̃ are 1; checked against
// the dense oracle at small sizes in tests/test_oracle_kat.py).
// xt_start / sigma2_start (optional; nullptr / ≤ 0 → X and init_sigma2):
// resume from a given EM state x̃ (in the frame the loop runs in: normalised
// when `normalize`) and σ² — the state is exactly (x̃, σ²), so a window of
// late iterations can be checked without replaying the whole run.
int orc_register_stream(const double* x_in, int64_t m, const double* y_in, int64_t n, int d,
                        double omega, double lambda_reg, int iterations, int normalize,
                        const double* u, const double* lam, const double* lam_num, int64_t k,
                        const double* xt_start, double sigma2_start,
                        double* out_x, double* sigma2_trace, int* iters_run,
                        double* sigma2_initial) {
  if (m == 0 || n == 0) return fail(kParameter, "register: empty point set");
  std::vector<double> x(m * d), y(n * d), center(d, 0.0);
  double scale = 1.0;
  int degen = 0;
  if (normalize) {
    int rc = orc_normalize_pair(x_in, m, y_in, n, d, x.data(), y.data(), center.data(), &scale,
                                &degen);
    if (rc) return rc;
  } else {
    std::memcpy(x.data(), x_in, sizeof(double) * m * d);
    std::memcpy(y.data(), y_in, sizeof(double) * n * d);
  }
  double sigma2 = 0.0;
  orc_init_sigma2(x.data(), m, y.data(), n, d, &sigma2);
  *sigma2_initial = sigma2;
  if (sigma2_start > 0.0) sigma2 = sigma2_start;
  std::vector<double> xt = x, pty(m * d), p1(m), var(m), resid(m * d), z(k * d), xn(m * d);
  if (xt_start) std::memcpy(xt.data(), xt_start, sizeof(double) * m * d);
  std::vector<int32_t> deg(m);
  int it = 0;
  for (; it < iterations; ++it) {
    int clamped = 0;
    int rc = orc_estep_stream(xt.data(), m, y.data(), n, d, omega, sigma2, pty.data(), p1.data(),
                              var.data(), deg.data(), nullptr, &clamped);
    if (rc) return fail(kNumeric, "register: iteration " + std::to_string(it) + ": " + g_err);
    for (int64_t i = 0; i < m * d; ++i) resid[i] = pty[i] - x[i];
    const double shift = lambda_reg * sigma2;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < k; ++j)
      for (int c = 0; c < d; ++c) {
        double acc = 0.0;
        for (int64_t r = 0; r < m; ++r) acc += u[j * m + r] * resid[c * m + r];
        z[c * k + j] = acc * lam_num[j] / (lam[j] + shift);
      }
    basis_times(u, m, k, z.data(), d, x.data(), xn.data());
    double tot = 0.0;
    for (int64_t r = 0; r < m; ++r) {
      double dd = 0.0, da = 0.0;
      for (int c = 0; c < d; ++c) {
        const double dl = xn[c * m + r] - xt[c * m + r];
        dd += dl * dl;
        da += dl * (pty[c * m + r] - xt[c * m + r]);
      }
      tot += var[r] - 2.0 * da + dd;
    }
    const double val = tot / (static_cast<double>(d) * static_cast<double>(m));
    if (val < -1e-8)
      return fail(kNumeric, "register: iteration " + std::to_string(it) +
                                ": update_sigma2: negative variance " + std::to_string(val));
    const double next = std::max(val, kSigma2Floor);
    sigma2_trace[it] = next;
    sigma2 = next;
    xt.swap(xn);
  }
  *iters_run = it;
  for (int c = 0; c < d; ++c)
    for (int64_t r = 0; r < m; ++r)
      out_x[c * m + r] = normalize ? xt[c * m + r] * scale + center[c] : xt[c * m + r];
  return kOk;
}

// Rows of Φ (kernel.hpp:31-47: exp(−max(|x_i|²+|x_j|²−2x_i·x_j, 0)/(2β²)),
// unit diagonal) for the model rows rows[0..nrows), column-major
// nrows × M.  The oracle's independent top-K basis (oracle.py topk_basis)
// and the eigen-residual checks form Φ·V block by block from these rows.
int orc_gram_rows(const double* x, int64_t m, int d, double beta, const int64_t* rows,
                  int64_t nrows, double* out) {
  if (beta <= 0.0) return fail(kParameter, "build_gram: beta must be positive");
  const double inv = 1.0 / (2.0 * beta * beta);
  std::vector<double> sq(m, 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int j = 0; j < d; ++j) sq[i] += at(x, m, i, j) * at(x, m, i, j);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < m; ++c) {
    for (int64_t q = 0; q < nrows; ++q) {
      const int64_t r = rows[q];
      double xy = 0.0;
      for (int j = 0; j < d; ++j) xy += at(x, m, r, j) * at(x, m, c, j);
      const double d2 = sq[r] + sq[c] - 2.0 * xy;
      out[c * nrows + q] = r == c ? 1.0 : std::exp(-std::max(d2, 0.0) * inv);
    }
  }
  return kOk;
}

void orc_make_cloud(int64_t m, int d, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t i = 0; i < m; ++i)
    for (int j = 0; j < d; ++j) out[j * m + i] = u(rng);
}

void orc_make_torus(int64_t m, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 2.0 * M_PI);
  for (int64_t i = 0; i < m; ++i) {
    const double a = u(rng), b = u(rng);
    out[0 * m + i] = (1.0 + 0.35 * std::cos(b)) * std::cos(a);
    out[1 * m + i] = (1.0 + 0.35 * std::cos(b)) * std::sin(a);
    out[2 * m + i] = 0.35 * std::sin(b);
  }
}

void orc_random_row_constrained(int64_t m, int64_t n, uint64_t seed, double* p) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      p[j * m + i] = u(rng);
      s += p[j * m + i];
    }
    for (int64_t j = 0; j < n; ++j) p[j * m + i] /= s;
  }
}

}  // extern "C"
