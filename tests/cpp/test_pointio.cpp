// Point-file I/O and run report of the drop-in header, restating the
// reference's tests (proj/tests/test_pointset.cpp:26-75 and the report keys
// of registration.hpp:178-204).  Host-only: no GPU needed.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

#include "fastcpd/fastcpd.hpp"

using namespace fastcpd;

static int g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    const bool ok_ = (cond);                                                     \
    std::printf("%s: %s (line %d)\n", ok_ ? "PASS" : "FAIL", #cond, __LINE__);  \
    if (!ok_) ++g_fail;                                                          \
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

static void write_text(const std::string& p, const std::string& s) {
  std::ofstream(p) << s;
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const std::string p = dir + "/fcpd_pointio.txt";

  // load_points reads whitespace rows in order
  write_text(p, "0 0\n1 1\n");
  PointSet ps = load_points(p);
  CHECK(ps.count() == 2 && ps.dim() == 2);
  CHECK(ps.pts(0, 0) == 0.0 && ps.pts(1, 1) == 1.0);

  // comments and commas
  write_text(p, "# header\n1 2 3\n");
  ps = load_points(p);
  CHECK(ps.count() == 1 && ps.dim() == 3);
  write_text(p, "1,2,3\n4, 5 ,6\n");
  ps = load_points(p);
  CHECK(ps.count() == 2 && ps.pts(1, 2) == 6.0);
  write_text(p, "\n  \n1 2 # trailing comment\n\n3 4\n");
  ps = load_points(p);
  CHECK(ps.count() == 2 && ps.pts(1, 0) == 3.0);

  // error paths
  write_text(p, "1 2\n3\n");
  CHECK(throws_as<DimensionError>([&] { load_points(p); }));
  write_text(p, "1 banana\n");
  CHECK(throws_as<ParseError>([&] { load_points(p); }));
  write_text(p, "1 inf\n");
  CHECK(throws_as<ParseError>([&] { load_points(p); }));
  write_text(p, "");
  CHECK(throws_as<ParseError>([&] { load_points(p); }));
  CHECK(throws_as<IoError>([&] { load_points("/nonexistent/dir/pts.txt"); }));
  write_text(p, "1 2\n3 4\n");
  CHECK(throws_as<DimensionError>([&] { load_points(p, 3); }));
  try {
    write_text(p, "1 2\n3 x4\n");
    load_points(p);
  } catch (const ParseError& e) {
    CHECK(std::string(e.what()).find(":2: malformed number 'x4'") != std::string::npos);
  }

  // write_points round-trips within 1e-12 (test_util.hpp make_cloud)
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  PointSet cloud;
  cloud.pts.resize(100, 3);
  for (Index i = 0; i < 100; ++i)
    for (Index j = 0; j < 3; ++j) cloud.pts(i, j) = u(rng);
  write_points(cloud, p);
  PointSet back = load_points(p);
  double err = 0.0;
  for (Index i = 0; i < 100; ++i)
    for (Index j = 0; j < 3; ++j) err = std::fmax(err, std::fabs(back.pts(i, j) - cloud.pts(i, j)));
  CHECK(back.count() == 100 && err <= 1e-12);
  CHECK(throws_as<IoError>([&] { write_points(cloud, "/nonexistent/dir/out.txt"); }));

  // run report: key=value lines, σ² trace last
  RegistrationConfig cfg;
  cfg.omega = 0.25;
  RegistrationResult res;
  res.sigma2_initial = 0.5;
  res.sigma2_trace = {0.4, 0.3};
  res.timing.t_total = 1.25;
  const std::string rp = dir + "/fcpd_report.txt";
  write_report(rp, cfg, res);
  std::ifstream in(rp);
  std::string all((std::istreambuf_iterator<char>(in)), {});
  for (const char* key : {"variant=fast\n", "omega=0.25\n", "beta=2\n", "lambda=10\n",
                          "iterations=100\n", "rank_fraction=0.1\n", "seed=0\n", "normalize=1\n",
                          "baseline_solver=dense LDLT factorization\n", "sigma2_initial=0.5\n",
                          "degenerate_rows=0\n", "sigma2_clamps=0\n", "t_total=1.25\n",
                          "sigma2[0]=0.4\n", "sigma2[1]=0.3\n"})
    CHECK(all.find(key) != std::string::npos);
  CHECK(throws_as<IoError>([&] { write_report("/nonexistent/dir/r.txt", cfg, res); }));

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
