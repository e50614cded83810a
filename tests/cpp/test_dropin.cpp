// Drop-in check: reference-style C++ test code (proj/tests/test_registration.cpp)
// compiled against include/fastcpd/fastcpd.hpp and run on the B200 engine.
// Exit code 0 = all checks passed; prints one line per check.
#include <cmath>
#include <cstdio>
#include <random>

#include "fastcpd/fastcpd.hpp"

using namespace fastcpd;

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    const bool ok_ = (cond);                                          \
    std::printf("%s: %s (line %d)\n", ok_ ? "PASS" : "FAIL", #cond, __LINE__); \
    if (!ok_) ++g_fail;                                               \
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

// test_util.hpp:13-37 restated
static PointSet make_cloud(Index m, Index d, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  PointSet ps;
  ps.pts.resize(m, d);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j) ps.pts(i, j) = u(rng);
  return ps;
}

static PointSet make_torus(Index m, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 2.0 * M_PI);
  PointSet ps;
  ps.pts.resize(m, 3);
  for (Index i = 0; i < m; ++i) {
    const double a = u(rng), b = u(rng);
    ps.pts(i, 0) = (1.0 + 0.35 * std::cos(b)) * std::cos(a);
    ps.pts(i, 1) = (1.0 + 0.35 * std::cos(b)) * std::sin(a);
    ps.pts(i, 2) = 0.35 * std::sin(b);
  }
  return ps;
}

int main() {
  {  // init_sigma2 cases (test_registration.cpp:13-27)
    PointSet x, y;
    x.pts.resize(1, 1);
    y.pts.resize(1, 1);
    y.pts(0, 0) = 2.0;
    CHECK(std::fabs(init_sigma2(x, y) - 4.0) <= 1e-14);
  }
  {  // self-registration converges (test_registration.cpp:29-42)
    PointSet x = make_torus(120, 52);
    RegistrationConfig cfg;
    cfg.iterations = 50;
    RegistrationResult res = register_pointsets(x, x, cfg);
    CHECK(res.sigma2_trace.size() == 50);
    double se = 0.0;
    for (Index i = 0; i < x.count(); ++i)
      for (Index j = 0; j < 3; ++j) {
        const double dlt = res.transformed.pts(i, j) - x.pts(i, j);
        se += dlt * dlt;
      }
    CHECK(std::sqrt(se / static_cast<double>(x.count())) <= 1e-3);
    bool mono = true;
    for (size_t i = 1; i < res.sigma2_trace.size(); ++i)
      mono = mono && res.sigma2_trace[i] <= res.sigma2_trace[i - 1] + 1e-12;
    CHECK(mono);
  }
  {  // zero iterations is the identity (:44-53)
    PointSet x = make_cloud(20, 2, 53), y = make_cloud(25, 2, 54);
    RegistrationConfig cfg;
    cfg.iterations = 0;
    RegistrationResult res = register_pointsets(x, y, cfg);
    double mx = 0.0, mw = 0.0;
    for (Index i = 0; i < 20; ++i)
      for (Index j = 0; j < 2; ++j) {
        mx = std::max(mx, std::fabs(res.transformed.pts(i, j) - x.pts(i, j)));
        mw = std::max(mw, std::fabs(res.coefficients.w(i, j)));
      }
    CHECK(mx <= 1e-12);
    CHECK(mw == 0.0);
    CHECK(res.sigma2_trace.empty());
  }
  {  // timing identities hold exactly (:55-70)
    PointSet x = make_cloud(60, 3, 55), y = make_cloud(60, 3, 56);
    for (SolverVariant v : {SolverVariant::fast, SolverVariant::fast_lowrank}) {
      RegistrationConfig cfg;
      cfg.iterations = 5;
      cfg.variant = v;
      const TimingBreakdown t = register_pointsets(x, y, cfg).timing;
      CHECK(t.t_f == t.t_eig + t.t_iter);
      CHECK(t.t_total == t.t_c + t.t_f + t.t_o);
    }
  }
  {  // bitwise-identical traces (:72-83)
    PointSet x = make_torus(80, 57), y = make_torus(90, 58);
    RegistrationConfig cfg;
    cfg.iterations = 15;
    RegistrationResult a = register_pointsets(x, y, cfg);
    RegistrationResult b = register_pointsets(x, y, cfg);
    CHECK(a.sigma2_trace == b.sigma2_trace);
  }
  {  // degenerate sizes (:85-97)
    PointSet x, y;
    x.pts.resize(1, 2);
    x.pts(0, 0) = 0.2;
    x.pts(0, 1) = 0.1;
    y.pts.resize(3, 2);
    y.pts(1, 0) = 1.0;
    y.pts(2, 1) = 1.0;
    for (SolverVariant v : {SolverVariant::fast, SolverVariant::fast_lowrank}) {
      RegistrationConfig cfg;
      cfg.iterations = 3;
      cfg.variant = v;
      RegistrationResult res = register_pointsets(x, y, cfg);
      CHECK(res.transformed.count() == 1 && res.sigma2_trace.size() == 3);
    }
  }
  {  // input validation (:99-106)
    PointSet x = make_cloud(5, 2, 59), y3 = make_cloud(5, 3, 60);
    RegistrationConfig cfg;
    CHECK(throws_as<DimensionError>([&] { register_pointsets(x, y3, cfg); }));
    cfg.iterations = -1;
    CHECK(throws_as<ParameterError>([&] { register_pointsets(x, x, cfg); }));
  }
  {  // correspondence on request is row-stochastic (acceptance.cpp:269-271)
    PointSet x = make_cloud(30, 3, 14), y = make_cloud(40, 3, 15);
    RegistrationConfig cfg;
    cfg.iterations = 5;
    cfg.want_correspondence = true;
    RegistrationResult res = register_pointsets(x, y, cfg);
    double worst = 0.0;
    for (Index i = 0; i < 30; ++i) {
      double s = 0.0;
      for (Index j = 0; j < 40; ++j) s += res.correspondence.p(i, j);
      worst = std::max(worst, std::fabs(s - 1.0));
    }
    CHECK(res.correspondence.row_constrained && worst <= 1e-10);
  }
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
