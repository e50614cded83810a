// The reference's L2 unit tests — proj/tests/test_correspondence.cpp,
// test_solvers.cpp (the fast solvers; the O(M³) cpd baselines are out of
// scope of the B200 path) and test_kernel.cpp — restated against the drop-in
// header include/fastcpd/fastcpd.hpp and run on the B200 through the C ABI.
// Same inputs (test_util.hpp generators restated: mt19937_64), same checks,
// same tolerances.  Exit code 0 = every check passed; one line per check.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <random>

#include "fastcpd/fastcpd.hpp"

using namespace fastcpd;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    const bool ok_ = (cond);                                                     \
    if (!ok_) std::printf("FAIL: %s (line %d)\n", #cond, __LINE__);             \
    ok_ ? ++g_pass : ++g_fail;                                                   \
  } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static bool approx(double a, double b, double eps = 1.19e-5) {  // doctest::Approx default scale
  return std::fabs(a - b) <= eps * (1.0 + std::max(std::fabs(a), std::fabs(b)));
}

// ---------------------------------------------------- test_util.hpp:13-52
static PointSet make_cloud(Index m, Index d, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  PointSet ps;
  ps.pts.resize(m, d);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j) ps.pts(i, j) = u(rng);
  return ps;
}

static Correspondence random_row_constrained(Index m, Index n, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  Correspondence c;
  c.p.resize(m, n);
  for (Index i = 0; i < m; ++i) {
    double s = 0.0;
    for (Index j = 0; j < n; ++j) s += (c.p(i, j) = u(rng));
    for (Index j = 0; j < n; ++j) c.p(i, j) /= s;
  }
  c.row_constrained = true;
  return c;
}

static PointSet pts(Index r, Index c, std::initializer_list<double> v) {  // row-major literal
  PointSet p;
  p.pts.resize(r, c);
  auto it = v.begin();
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) p.pts(i, j) = *it++;
  return p;
}

// ------------------------------------------------ small dense helpers (host)
static Matrix mul(const Matrix& a, const Matrix& b, bool ta = false, bool tb = false) {
  const Index n = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
  const Index m = tb ? b.rows() : b.cols();
  Matrix c(n, m);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < m; ++j) {
      double s = 0.0;
      for (Index q = 0; q < k; ++q) s += (ta ? a(q, i) : a(i, q)) * (tb ? b(j, q) : b(q, j));
      c(i, j) = s;
    }
  return c;
}
static Matrix lincomb(const Matrix& a, double fa, const Matrix& b, double fb) {
  Matrix c(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c(i, j) = fa * a(i, j) + fb * b(i, j);
  return c;
}
static double norm(const Matrix& a) {
  double s = 0.0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s += a(i, j) * a(i, j);
  return std::sqrt(s);
}
static double maxabs(const Matrix& a) {
  double s = 0.0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s = std::max(s, std::fabs(a(i, j)));
  return s;
}
static Matrix diag_scale(const Matrix& u, const Vector& l) {  // U diag(l)
  Matrix c = u;
  for (Index j = 0; j < u.cols(); ++j)
    for (Index i = 0; i < u.rows(); ++i) c(i, j) *= l(j);
  return c;
}
static Matrix eye(Index n) {
  Matrix e(n, n);
  for (Index i = 0; i < n; ++i) e(i, i) = 1.0;
  return e;
}
// dense SPD solve by Cholesky (the reference's LDLT oracle, host fp64)
static Matrix spd_solve(Matrix a, Matrix b) {
  const Index n = a.rows();
  for (Index j = 0; j < n; ++j) {
    double d = a(j, j);
    for (Index k = 0; k < j; ++k) d -= a(j, k) * a(j, k);
    a(j, j) = std::sqrt(d);
    for (Index i = j + 1; i < n; ++i) {
      double s = a(i, j);
      for (Index k = 0; k < j; ++k) s -= a(i, k) * a(j, k);
      a(i, j) = s / a(j, j);
    }
  }
  for (Index c = 0; c < b.cols(); ++c) {
    for (Index i = 0; i < n; ++i) {
      double s = b(i, c);
      for (Index k = 0; k < i; ++k) s -= a(i, k) * b(k, c);
      b(i, c) = s / a(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = b(i, c);
      for (Index k = i + 1; k < n; ++k) s -= a(k, i) * b(k, c);
      b(i, c) = s / a(i, i);
    }
  }
  return b;
}

// ===================================================== test_correspondence.cpp
static void correspondence_tests() {
  {  // single component takes all mass (:10-16)
    PointSet x = pts(1, 2, {0, 0});
    PointSet y = make_cloud(5, 2, 1);
    Correspondence c = posterior(x, y, GmmParams{0.0, 0.5});
    for (Index j = 0; j < 5; ++j) CHECK(approx(c.p(0, j), 1.0, 1e-14));
  }
  {  // equidistant symmetry (:18-24)
    PointSet x = pts(2, 2, {-1, 0, 1, 0});
    PointSet y = pts(1, 2, {0, 0.3});
    Correspondence c = posterior(x, y, GmmParams{0.0, 0.25});
    CHECK(approx(c.p(0, 0), 0.5));
    CHECK(approx(c.p(1, 0), 0.5));
  }
  {  // scalar value with the outlier term (:26-35)
    Correspondence c = posterior(pts(1, 1, {0}), pts(1, 1, {1}), GmmParams{0.5, 1.0});
    const double e = std::exp(-0.5);
    CHECK(approx(c.p(0, 0), e / (e + std::sqrt(2.0 * M_PI)), 1e-12));
    CHECK(approx(c.p(0, 0), 0.1948, 1e-3));
  }
  {  // parameter handling (:37-45)
    PointSet x = make_cloud(3, 2, 2), y = make_cloud(4, 2, 3);
    CHECK(throws_as<ParameterError>([&] { posterior(x, y, GmmParams{1.0, 1.0}); }));
    CHECK(throws_as<ParameterError>([&] { posterior(x, y, GmmParams{-0.1, 1.0}); }));
    CHECK(posterior(x, y, GmmParams{0.5, 1e-30}).sigma2_clamped);
  }
  {  // column sums (:47-60)
    PointSet x = make_cloud(8, 3, 4), y = make_cloud(6, 3, 5);
    Vector s0 = posterior(x, y, GmmParams{0.0, 0.3}).col_sums();
    for (Index j = 0; j < 6; ++j) CHECK(approx(s0(j), 1.0, 1e-10));
    Correspondence c = posterior(x, y, GmmParams{0.7, 0.3});
    Vector s = c.col_sums();
    for (Index j = 0; j < 6; ++j) CHECK(s(j) <= 1.0 + 1e-10);
    double mn = 1e300, mx = -1e300;
    for (Index j = 0; j < 6; ++j)
      for (Index i = 0; i < 8; ++i) mn = std::min(mn, c.p(i, j)), mx = std::max(mx, c.p(i, j));
    CHECK(mn >= 0.0);
    CHECK(mx <= 1.0);
  }
  {  // agrees with the unshifted formula (:62-83)
    PointSet x = make_cloud(5, 2, 6), y = make_cloud(7, 2, 7);
    const double omega = 0.3, sigma2 = 0.4;
    Correspondence c = posterior(x, y, GmmParams{omega, sigma2});
    const double cc = 2.0 * M_PI * sigma2 * (omega / (1.0 - omega)) * (5.0 / 7.0);
    auto d2 = [&](Index j, Index i) {
      double s = 0;
      for (Index k = 0; k < 2; ++k) s += (y.pts(j, k) - x.pts(i, k)) * (y.pts(j, k) - x.pts(i, k));
      return s;
    };
    for (Index j = 0; j < 7; ++j) {
      double denom = cc;
      for (Index i = 0; i < 5; ++i) denom += std::exp(-d2(j, i) / (2.0 * sigma2));
      for (Index i = 0; i < 5; ++i)
        CHECK(approx(c.p(i, j), std::exp(-d2(j, i) / (2.0 * sigma2)) / denom, 1e-12));
    }
  }
  {  // enforce_row_constraint: normalise, fall back, idempotent (:85-106)
    Correspondence raw;
    raw.p.resize(2, 2);
    raw.p(0, 0) = 0.2, raw.p(0, 1) = 0.2, raw.p(1, 0) = 0.0, raw.p(1, 1) = 0.5;
    Correspondence c = enforce_row_constraint(raw);
    CHECK(c.row_constrained);
    CHECK(approx(c.p(0, 0), 0.5));
    CHECK(approx(c.p(0, 1), 0.5));
    CHECK(c.p(1, 0) == 0.0);
    CHECK(approx(c.p(1, 1), 1.0));
    CHECK(c.degenerate_rows.empty());
    Correspondence again = enforce_row_constraint(c);
    CHECK(maxabs(lincomb(again.p, 1.0, c.p, -1.0)) == 0.0);
    Correspondence zero;
    zero.p = Matrix::Zero(1, 4);
    Correspondence fixed = enforce_row_constraint(zero);
    CHECK(fixed.degenerate_rows.size() == 1 && fixed.degenerate_rows[0] == 0);
    for (Index j = 0; j < 4; ++j) CHECK(fixed.p(0, j) == 0.25);
  }
  {  // estimated_targets cases and convexity (:108-139)
    PointSet y = pts(2, 2, {0, 0, 2, 0});
    Correspondence ident;
    ident.p = eye(2);
    ident.row_constrained = true;
    CHECK(maxabs(lincomb(estimated_targets(ident, y).pts, 1.0, y.pts, -1.0)) == 0.0);
    Correspondence uniform;
    uniform.p = Matrix(1, 2);
    uniform.p(0, 0) = uniform.p(0, 1) = 0.5;
    CHECK(approx(estimated_targets(uniform, y).pts(0, 0), 1.0));
    Correspondence weighted;
    weighted.p = Matrix(1, 2);
    weighted.p(0, 0) = 0.25, weighted.p(0, 1) = 0.75;
    CHECK(approx(estimated_targets(weighted, pts(2, 2, {0, 0, 4, 0})).pts(0, 0), 3.0));
    PointSet ybig = make_cloud(9, 3, 8);
    PointSet t = estimated_targets(random_row_constrained(12, 9, 9), ybig);
    for (Index j = 0; j < 3; ++j) {
      double ymn = 1e300, ymx = -1e300, tmn = 1e300, tmx = -1e300;
      for (Index i = 0; i < 9; ++i) ymn = std::min(ymn, ybig.pts(i, j)), ymx = std::max(ymx, ybig.pts(i, j));
      for (Index i = 0; i < 12; ++i) tmn = std::min(tmn, t.pts(i, j)), tmx = std::max(tmx, t.pts(i, j));
      CHECK(tmn >= ymn - 1e-12);
      CHECK(tmx <= ymx + 1e-12);
    }
    CHECK(throws_as<ParameterError>([&] { estimated_targets(ident, make_cloud(5, 2, 1)); }));
  }
}

// ========================================================= test_solvers.cpp
struct Instance {
  PointSet x, y;
  GramKernel gram;
  SpectralBasis basis;  // full rank
  Correspondence p;     // row constrained
  double lambda_reg = 10.0, sigma2 = 0.3;
};
static Instance make_instance(Index m, Index n, Index d, unsigned long seed) {
  Instance inst;
  inst.x = make_cloud(m, d, seed);
  inst.y = make_cloud(n, d, seed + 1);
  inst.gram = build_gram(inst.x, 2.0);
  inst.basis = eigendecompose(inst.gram, m);
  inst.p = random_row_constrained(m, n, seed + 2);
  return inst;
}
static Matrix residual_of(const Instance& inst) {
  return lincomb(mul(inst.p.p, inst.y.pts), 1.0, inst.x.pts, -1.0);
}

static void solver_tests() {
  {  // zero residual and the scalar case (:35-49)
    Instance inst = make_instance(6, 6, 2, 20);
    CHECK(maxabs(solve_fast(inst.basis, 10.0, 0.3, Matrix::Zero(6, 2)).w) == 0.0);
    SpectralBasis b1;
    b1.u = Matrix(1, 1);
    b1.u(0, 0) = 1.0;
    b1.lambda.resize(1);
    b1.lambda(0) = 1.0;
    Matrix r(1, 1);
    r(0, 0) = 0.8;
    CHECK(approx(solve_fast(b1, 2.0, 0.25, r).w(0, 0), 0.8 / (1.0 + 2.0 * 0.25), 1e-14));
  }
  {  // matches a dense factorisation of (Φ + λσ² I) W = R (:51-68)
    Instance inst = make_instance(100, 80, 3, 21);
    Matrix residual = residual_of(inst);
    Coefficients fast = solve_fast(inst.basis, inst.lambda_reg, inst.sigma2, residual);
    Matrix a = inst.gram.phi;
    for (Index i = 0; i < 100; ++i) a(i, i) += inst.lambda_reg * inst.sigma2;
    Matrix dense = spd_solve(a, residual);
    CHECK(norm(lincomb(fast.w, 1.0, dense, -1.0)) <= 1e-8 * norm(dense));
    CHECK(norm(lincomb(mul(a, fast.w), 1.0, residual, -1.0)) <= 1e-8 * norm(residual));
    Coefficients scaled = solve_fast(inst.basis, inst.lambda_reg, inst.sigma2,
                                     lincomb(residual, 3.5, residual, 0.0));
    CHECK(norm(lincomb(scaled.w, 1.0, fast.w, -3.5)) <= 1e-10 * norm(scaled.w));
  }
  {  // low rank at K = M reproduces solve_fast (:70-79)
    Instance inst = make_instance(40, 30, 2, 22);
    Matrix residual = residual_of(inst);
    Coefficients full = solve_fast(inst.basis, inst.lambda_reg, inst.sigma2, residual);
    Coefficients lr = solve_fast_lowrank(inst.basis, inst.lambda_reg, inst.sigma2, residual);
    CHECK(maxabs(lincomb(full.w, 1.0, lr.w, -1.0)) <= 1e-12);
    CHECK(maxabs(solve_fast_lowrank(inst.basis, 10.0, 0.3, Matrix::Zero(40, 2)).w) == 0.0);
  }
  {  // truncated system within the basis span (:81-102)
    Instance inst = make_instance(100, 100, 3, 23);
    SpectralBasis trunc = eigendecompose(inst.gram, 10);
    Matrix residual = residual_of(inst);
    Coefficients lr = solve_fast_lowrank(trunc, inst.lambda_reg, inst.sigma2, residual);
    Matrix a = mul(diag_scale(trunc.u, trunc.lambda), trunc.u, false, true);
    for (Index i = 0; i < 100; ++i) a(i, i) += inst.lambda_reg * inst.sigma2;
    Matrix small = mul(trunc.u, mul(a, trunc.u), true, false);  // Λ + λσ² I
    Matrix z = spd_solve(small, mul(trunc.u, residual, true, false));
    Matrix dense = mul(trunc.u, z);
    CHECK(norm(lincomb(lr.w, 1.0, dense, -1.0)) <= 1e-8 * norm(dense));
    CHECK(norm(lincomb(lr.w, 1.0, mul(trunc.u, mul(trunc.u, lr.w, true, false)), -1.0)) <=
          1e-10 * norm(lr.w));
    CHECK(norm(mul(trunc.u, lincomb(mul(a, lr.w), 1.0, residual, -1.0), true, false)) <=
          1e-8 * norm(residual));
  }
  {  // apply_transform variants (:151-190)
    Instance inst = make_instance(30, 30, 3, 35);
    Coefficients zero{Matrix::Zero(30, 3)};
    CHECK(maxabs(lincomb(apply_transform(inst.x, inst.gram, zero).pts, 1.0, inst.x.pts, -1.0)) ==
          0.0);
    PointSet x1 = pts(1, 2, {0.1, 0.2});
    GramKernel g1 = build_gram(x1, 2.0);
    Coefficients w1{pts(1, 2, {0.3, -0.4}).pts};
    PointSet t1 = apply_transform(x1, g1, w1);
    CHECK(approx(t1.pts(0, 0), 0.4));
    CHECK(approx(t1.pts(0, 1), -0.2));
    Coefficients w{lincomb(make_cloud(30, 3, 36).pts, 0.1, make_cloud(30, 3, 36).pts, 0.0)};
    PointSet t = apply_transform(inst.x, inst.gram, w);
    for (Index i = 0; i < 30; ++i) {
      double acc[3] = {inst.x.pts(i, 0), inst.x.pts(i, 1), inst.x.pts(i, 2)};
      for (Index k = 0; k < 30; ++k) {
        double d2 = 0.0;
        for (Index c = 0; c < 3; ++c)
          d2 += (inst.x.pts(i, c) - inst.x.pts(k, c)) * (inst.x.pts(i, c) - inst.x.pts(k, c));
        for (Index c = 0; c < 3; ++c) acc[c] += w.w(k, c) * std::exp(-d2 / 8.0);
      }
      double e = 0.0;
      for (Index c = 0; c < 3; ++c) e = std::max(e, std::fabs(t.pts(i, c) - acc[c]));
      CHECK(e <= 1e-10);
    }
    CHECK(maxabs(lincomb(apply_transform_lowrank(inst.x, inst.basis, w).pts, 1.0, t.pts, -1.0)) <=
          1e-10);
    SpectralBasis trunc = eigendecompose(inst.gram, 5);
    Matrix recon = mul(diag_scale(trunc.u, trunc.lambda), trunc.u, false, true);
    PointSet tl = apply_transform_lowrank(inst.x, trunc, w);
    CHECK(maxabs(lincomb(tl.pts, 1.0, lincomb(inst.x.pts, 1.0, mul(recon, w.w), 1.0), -1.0)) <=
          1e-10);
    CHECK(maxabs(lincomb(apply_transform_lowrank(inst.x, trunc, zero).pts, 1.0, inst.x.pts,
                         -1.0)) == 0.0);
    CHECK(throws_as<ParameterError>([&] { apply_transform(x1, inst.gram, w1); }));
  }
  {  // update_sigma2: trace form vs the double sum (:192-223)
    PointSet y = make_cloud(10, 2, 40);
    Correspondence ident;
    ident.p = eye(10);
    ident.row_constrained = true;
    CHECK(update_sigma2(y, ident, y) == kSigma2Floor);
    Correspondence p1;
    p1.p = Matrix(1, 1);
    p1.p(0, 0) = 1.0;
    p1.row_constrained = true;
    CHECK(approx(update_sigma2(pts(1, 1, {2}), p1, pts(1, 1, {0})), 4.0, 1e-14));
    PointSet yb = make_cloud(30, 3, 41), xb = make_cloud(20, 3, 42);
    Correspondence p = random_row_constrained(20, 30, 43);
    const double trace = update_sigma2(yb, p, xb);
    double dbl = 0.0;
    for (Index i = 0; i < 20; ++i)
      for (Index j = 0; j < 30; ++j) {
        double d2 = 0.0;
        for (Index c = 0; c < 3; ++c) d2 += (yb.pts(j, c) - xb.pts(i, c)) * (yb.pts(j, c) - xb.pts(i, c));
        dbl += p.p(i, j) * d2;
      }
    dbl /= 3.0 * 20.0;
    CHECK(approx(trace, dbl, 1e-10));
    Correspondence unconstrained = p;
    unconstrained.row_constrained = false;
    CHECK(throws_as<ParameterError>([&] { update_sigma2(yb, unconstrained, xb); }));
  }
}

// ========================================================== test_kernel.cpp
static void kernel_tests() {
  {  // build_gram scalar cases (:11-26)
    CHECK(build_gram(pts(1, 2, {0.3, -0.7}), 2.0).phi(0, 0) == 1.0);
    GramKernel k2 = build_gram(pts(2, 2, {1, 1, 1, 1}), 2.0);
    CHECK(approx(std::min(std::min(k2.phi(0, 0), k2.phi(0, 1)), k2.phi(1, 0)), 1.0));
    PointSet line = pts(2, 1, {0, 2});
    CHECK(approx(build_gram(line, 2.0).phi(0, 1), std::exp(-0.5)));
    CHECK(throws_as<ParameterError>([&] { build_gram(line, 0.0); }));
    CHECK(throws_as<ParameterError>([&] { build_gram(line, -1.0); }));
  }
  {  // Gram invariants (:28-38)
    GramKernel k = build_gram(make_cloud(60, 3, 11), 2.0);
    double asym = 0.0, dmin = 1e300, mn = 1e300, mx = -1e300;
    for (Index i = 0; i < 60; ++i) {
      dmin = std::min(dmin, k.phi(i, i));
      for (Index j = 0; j < 60; ++j) {
        asym = std::max(asym, std::fabs(k.phi(i, j) - k.phi(j, i)));
        mn = std::min(mn, k.phi(i, j));
        mx = std::max(mx, k.phi(i, j));
      }
    }
    CHECK(asym == 0.0);
    CHECK(dmin == 1.0);
    CHECK(mn > 0.0);
    CHECK(mx <= 1.0);
    CHECK(eigendecompose(k, 60).lambda.minCoeff() >= -1e-8 * 60);
  }
  {  // near-identity Gram (:40-51)
    SpectralBasis b = eigendecompose(build_gram(pts(4, 1, {0, 1e5, 2e5, 3e5}), 2.0), 4);
    for (Index i = 0; i < 4; ++i) CHECK(approx(b.lambda(i), 1.0, 1e-12));
    CHECK(maxabs(lincomb(mul(b.u, b.u, true, false), 1.0, eye(4), -1.0)) <= 1e-8);
  }
  {  // duplicate points give {2, 0} (:53-59)
    SpectralBasis b = eigendecompose(build_gram(pts(2, 2, {1, 1, 1, 1}), 2.0), 2);
    CHECK(approx(b.lambda(0), 2.0));
    CHECK(approx(b.lambda(1), 0.0));
  }
  {  // full-rank reconstruction and orthonormality (:61-75)
    GramKernel k = build_gram(make_cloud(50, 3, 3), 2.0);
    SpectralBasis b = eigendecompose(k, 50);
    CHECK(maxabs(lincomb(mul(b.u, b.u, true, false), 1.0, eye(50), -1.0)) <= 1e-8);
    Matrix recon = mul(diag_scale(b.u, b.lambda), b.u, false, true);
    CHECK(norm(lincomb(recon, 1.0, k.phi, -1.0)) <= 1e-6 * norm(k.phi));
    bool desc = true;
    for (Index i = 0; i + 1 < 50; ++i) desc = desc && b.lambda(i) >= b.lambda(i + 1);
    CHECK(desc);
    CHECK(throws_as<ParameterError>([&] { eigendecompose(k, 0); }));
    CHECK(throws_as<ParameterError>([&] { eigendecompose(k, 51); }));
  }
  {  // reconstruction error = the dropped tail (:77-96)
    GramKernel k = build_gram(make_cloud(50, 2, 9), 2.0);
    SpectralBasis full = eigendecompose(k, 50);
    double prev = 1e300;
    for (Index kk : {1, 10, 25, 50}) {
      const double err = lowrank_reconstruction_error(eigendecompose(k, kk), k);
      double tail = 0.0;
      for (Index i = kk; i < 50; ++i) tail += full.lambda(i) * full.lambda(i);
      tail = std::sqrt(tail);
      if (tail > 0.0)
        CHECK(approx(err, tail, 1e-8));
      else
        CHECK(err <= 1e-6 * norm(k.phi));
      CHECK(err <= prev + 1e-12);
      prev = err;
    }
  }
  {  // spectral cache round trip (:98-110)
    SpectralBasis b = eigendecompose(build_gram(make_cloud(20, 3, 5), 2.0), 7);
    const std::string path = (std::filesystem::temp_directory_path() / "fcpd_l2_cache.bin").string();
    save_spectral_cache(path, b, 2.0);
    double beta = 0.0;
    SpectralBasis back = load_spectral_cache(path, &beta);
    CHECK(beta == 2.0);
    CHECK(back.rank() == 7);
    CHECK(maxabs(lincomb(back.u, 1.0, b.u, -1.0)) == 0.0);
    double dl = 0.0;
    for (Index i = 0; i < 7; ++i) dl = std::max(dl, std::fabs(back.lambda(i) - b.lambda(i)));
    CHECK(dl == 0.0);
    std::remove(path.c_str());
  }
  {  // normalize_pair (test_pointset.cpp:77-113)
    PointSet x = pts(2, 2, {0, 0, 2, 0}), y = pts(1, 2, {1, 3});
    auto [xn, yn, rec] = normalize_pair(x, y);
    CHECK(approx(rec.center(0), 1.0) && approx(rec.center(1), 1.0));
    CHECK(approx(rec.scale, 2.0) && !rec.degenerate);
    CHECK(approx(yn.pts(0, 1), 1.0));
    CHECK(maxabs(lincomb(rec.invert(xn).pts, 1.0, x.pts, -1.0)) <= 1e-15);
    auto [xd, yd, rd] = normalize_pair(pts(1, 2, {1, 1}), pts(1, 2, {1, 1}));
    CHECK(rd.degenerate && rd.scale == 1.0);
    CHECK(throws_as<DimensionError>([&] { normalize_pair(pts(1, 2, {0, 0}), pts(1, 1, {0})); }));
    CHECK(throws_as<ParameterError>([&] { normalize_pair(PointSet{}, pts(1, 1, {0})); }));
  }
}

int main() {
  try {
    correspondence_tests();
    solver_tests();
    kernel_tests();
  } catch (const std::exception& e) {
    std::printf("FAIL: uncaught %s\n", e.what());
    return 2;
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
