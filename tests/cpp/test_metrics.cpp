// Benchmark-harness helpers of the drop-in header (rmse, subsample,
// random_affine, make_bench_pair, the bench CSV, bench_plot), restating the
// host-only cases of the reference's proj/tests/test_metrics.cpp:12-131.  No GPU:
// BenchRecords are built by hand instead of through run_benchmark.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
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

static PointSet make_cloud(Index m, Index d, unsigned long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  PointSet ps;
  ps.pts.resize(m, d);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j) ps.pts(i, j) = u(rng);
  return ps;
}

static std::string slurp(const std::string& p) {
  std::ifstream f(p);
  return std::string((std::istreambuf_iterator<char>(f)), {});
}

static bool near(double a, double b, double rel) {
  return std::fabs(a - b) <= rel * std::fmax(1.0, std::fabs(b));
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";

  // rmse exact values (test_metrics.cpp:12-31)
  PointSet t;
  t.pts.resize(2, 2);
  t.pts(0, 0) = 0, t.pts(0, 1) = 0, t.pts(1, 0) = 1, t.pts(1, 1) = 1;
  Truth truth{{0, {0.0, 0.0}}, {1, {1.0, 1.0}}};
  CHECK(rmse(t, truth) == 0.0);
  Truth offset{{0, {3.0, 4.0}}};
  CHECK(near(rmse(t, offset), 5.0, 1e-14));
  PointSet t2;
  t2.pts.resize(2, 1);
  t2.pts(0, 0) = 0, t2.pts(1, 0) = 0;
  Truth two{{0, {0.0}}, {1, {2.0}}};
  CHECK(near(rmse(t2, two), std::sqrt(2.0), 1e-14));
  CHECK(throws_as<ParameterError>([&] { rmse(t, Truth{}); }));
  CHECK(throws_as<ParameterError>([&] { rmse(t, Truth{{5, {0.0, 0.0}}}); }));
  CHECK(throws_as<DimensionError>([&] { rmse(t, Truth{{0, {0.0}}}); }));

  // rmse invariant under a consistent permutation (test_metrics.cpp:33-46)
  {
    PointSet c = make_cloud(10, 3, 90);
    Truth tr, rtr;
    for (Index i = 0; i < 10; ++i) tr[i] = {c.pts(i, 0) + 0.01 * (i + 1), c.pts(i, 1), c.pts(i, 2)};
    PointSet rev;
    rev.pts.resize(10, 3);
    for (Index i = 0; i < 10; ++i)
      for (Index j = 0; j < 3; ++j) rev.pts(9 - i, j) = c.pts(i, j);
    for (Index i = 0; i < 10; ++i) rtr[9 - i] = tr[i];
    CHECK(near(rmse(rev, rtr), rmse(c, tr), 1e-14));
  }

  // subsample: exact size, seed-deterministic, source order (test_metrics.cpp:48-56)
  {
    PointSet src = make_cloud(200, 3, 91);
    PointSet a = subsample(src, 50, 7), b = subsample(src, 50, 7), c = subsample(src, 50, 8);
    CHECK(a.count() == 50 && a.dim() == 3);
    double diff = 0.0, diff_c = 0.0;
    for (Index i = 0; i < 50; ++i)
      for (Index j = 0; j < 3; ++j) {
        diff = std::fmax(diff, std::fabs(a.pts(i, j) - b.pts(i, j)));
        diff_c = std::fmax(diff_c, std::fabs(a.pts(i, j) - c.pts(i, j)));
      }
    CHECK(diff == 0.0);
    CHECK(diff_c > 0.0);
    CHECK(throws_as<ParameterError>([&] { subsample(src, 0, 7); }));
    CHECK(throws_as<ParameterError>([&] { subsample(src, 201, 7); }));
  }

  // random_affine stays mild (test_metrics.cpp:58-64): displacement ≤ 0.6
  for (Index d : {2, 3}) {
    PointSet src = make_cloud(300, d, 92);
    PointSet w = random_affine(src, 93);
    double worst = 0.0, moved = 0.0;
    for (Index i = 0; i < src.count(); ++i) {
      double r2 = 0.0;
      for (Index j = 0; j < d; ++j) r2 += (w.pts(i, j) - src.pts(i, j)) * (w.pts(i, j) - src.pts(i, j));
      worst = std::fmax(worst, std::sqrt(r2));
      moved += r2;
    }
    CHECK(worst <= 0.6);
    CHECK(moved > 0.0);
  }

  // make_bench_pair: scene in [-1, 1], truth = scene rows, model ≠ scene
  {
    PointSet src = make_cloud(120, 3, 94);
    DegradedPair p = make_bench_pair(src, 40, 11);
    CHECK(p.model.count() == 40 && p.scene.count() == 40 && p.truth.size() == 40);
    double amax = 0.0;
    for (Index i = 0; i < 40; ++i)
      for (Index j = 0; j < 3; ++j) amax = std::fmax(amax, std::fabs(p.scene.pts(i, j)));
    CHECK(near(amax, 1.0, 1e-12));
    CHECK(rmse(p.scene, p.truth) == 0.0);
    CHECK(rmse(p.model, p.truth) > 0.0);
  }

  // bench CSV: schema, rounding identities, byte-stable round trip, failed
  // cells as rmse −1 (test_metrics.cpp:84-109)
  {
    std::vector<BenchRecord> recs;
    const SolverVariant vs[2] = {SolverVariant::fast, SolverVariant::fast_lowrank};
    for (int k = 0; k < 4; ++k) {
      BenchRecord r;
      r.m = 30 + 10 * k, r.n = 30 + 10 * k;
      r.variant = vs[k % 2];
      r.timing.t_c = 1.23456789e-3 * (k + 1);
      r.timing.t_eig = 2.0000004e-3 * (k + 1);
      r.timing.t_iter = 0.1234565 * (k + 1);
      r.timing.t_o = 7.77e-7;
      r.timing.t_f = r.timing.t_eig + r.timing.t_iter;
      r.timing.t_total = r.timing.t_c + r.timing.t_f + r.timing.t_o;
      r.rmse = 1e-4 * (k + 1);
      r.iterations = 2;
      r.failed = (k == 3);
      recs.push_back(r);
    }
    const std::string p1 = dir + "/fcpd_bench1.csv", p2 = dir + "/fcpd_bench2.csv";
    write_bench_csv(recs, p1);
    const std::string s1 = slurp(p1);
    CHECK(s1.rfind(std::string(kBenchCsvHeader) + "\n", 0) == 0);
    auto back = load_bench_csv(p1);
    CHECK(back.size() == recs.size());
    write_bench_csv(back, p2);
    CHECK(s1 == slurp(p2));
    bool ident = true;
    for (const auto& r : back) {
      ident = ident && near(r.timing.t_f, r.timing.t_eig + r.timing.t_iter, 1e-12);
      ident = ident && near(r.timing.t_total, r.timing.t_c + r.timing.t_f + r.timing.t_o, 1e-12);
    }
    CHECK(ident);
    CHECK(back[1].variant == SolverVariant::fast_lowrank && back[1].m == 40);
    CHECK(!back[0].failed && back[3].failed && back[3].rmse == -1.0);
    CHECK(back[2].iterations == 2);

    std::ofstream(dir + "/fcpd_bad.csv") << "1 2 3\n";
    CHECK(throws_as<ParseError>([&] { load_bench_csv(dir + "/fcpd_bad.csv"); }));
    std::ofstream(dir + "/fcpd_bad2.csv") << kBenchCsvHeader << "\n1,2,fast,0\n";
    CHECK(throws_as<ParseError>([&] { load_bench_csv(dir + "/fcpd_bad2.csv"); }));
    CHECK(throws_as<IoError>([&] { load_bench_csv("/nonexistent/dir/b.csv"); }));
    CHECK(throws_as<IoError>([&] { write_bench_csv(recs, "/nonexistent/dir/b.csv"); }));
  }

  // bench_plot: deterministic, one path per variant with data, labelled axes,
  // an empty shell without data (test_metrics.cpp:111-131)
  {
    std::vector<BenchRecord> recs;
    const SolverVariant vs[3] = {SolverVariant::fast, SolverVariant::fast_lowrank,
                                 SolverVariant::cpd};
    for (int v = 0; v < 3; ++v)
      for (Index m : {30, 50, 80}) {
        BenchRecord r;
        r.m = r.n = m;
        r.variant = vs[v];
        r.timing.t_iter = 1e-3 * m * (v + 1);
        r.failed = (v == 2);  // the device path records cpd as failed cells
        recs.push_back(r);
      }
    const std::string a = bench_plot(recs), b = bench_plot(recs);
    CHECK(a == b);
    size_t paths = 0;
    for (size_t pos = a.find("<path d=\"M "); pos != std::string::npos;
         pos = a.find("<path d=\"M ", pos + 1))
      ++paths;
    CHECK(paths == 2);
    CHECK(a.find("M (log scale)") != std::string::npos);
    CHECK(a.find("seconds") != std::string::npos);
    CHECK(a.rfind("<svg", 0) == 0 && a.find("</svg>") != std::string::npos);
    const std::string e = bench_plot({});
    CHECK(e.find("<svg") != std::string::npos && e.find("<path d=\"M ") == std::string::npos);
    CHECK(throws_as<IoError>([&] { write_text_file(a, "/nonexistent/dir/p.svg"); }));
  }

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
