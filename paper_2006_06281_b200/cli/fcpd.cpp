// fcpd — command-line registration on the B200 engine.
//
// The `register` subcommand of the reference CLI (proj/tools/fcpd.cpp:56-83,
// flags :20-42, :198-215) over the drop-in C++ API: read two point files,
// register the model onto the scene on the GPU, write the transformed model
// and the key=value run report.  Same flags and defaults (ω=0.7, β=2,
// λ=10, 100 iterations, variant fast, rank fraction 0.1, seed 0).
// --svg writes a plain scatter overlay of the first two coordinates
// (registered model over scene).  `bench` sweeps sizes × variants in the
// reference's CSV schema (+ its t_iter chart); `plot` re-renders a CSV.
// Not provided: degrade.
//
//   fcpd register MODEL SCENE [--omega W] [--beta B] [--lambda L] [--iters N]
//        [--variant fast|fast-lowrank] [--rank-fraction F] [--seed S]
//        [--no-normalize] [--swap] [--early-stop] [--out FILE] [--report FILE]
//        [--svg FILE] [--device D]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "fastcpd/fastcpd.hpp"

namespace fc = fastcpd;

namespace {

int usage(const char* prog, int code) {
  std::fprintf(code ? stderr : stdout,
               "usage: %s register MODEL SCENE [--omega W] [--beta B] [--lambda L] [--iters N]\n"
               "          [--variant fast|fast-lowrank] [--rank-fraction F] [--seed S]\n"
               "          [--no-normalize] [--swap] [--early-stop] [--out FILE]\n"
               "          [--report FILE] [--svg FILE] [--device D]\n"
               "       %s bench [SOURCE | --synthetic] --sizes M1,M2,... [--variants fast,...]\n"
               "          [--iters N] [--seed S] [--csv FILE] [--svg FILE] [--device D]\n"
               "       %s plot BENCH_CSV [--out FILE]\n",
               prog, prog, prog);
  return code;
}

double to_double(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const double d = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw fc::ParameterError(flag + ": not a number: " + v);
  return d;
}

long to_long(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const long d = std::strtol(v.c_str(), &end, 10);
  if (v.empty() || *end) throw fc::ParameterError(flag + ": not an integer: " + v);
  return d;
}

// Scatter overlay of the first two coordinates: scene (red) under the
// registered model (blue), both in the scene's bounding box.
void write_overlay_svg(const fc::PointSet& moved, const fc::PointSet& scene,
                       const std::string& path) {
  const int w = 640, h = 640, pad = 20;
  double lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300};
  for (const fc::PointSet* ps : {&moved, &scene})
    for (fc::Index i = 0; i < ps->count(); ++i)
      for (int j = 0; j < 2; ++j) {
        const double v = ps->dim() > j ? ps->pts(i, j) : 0.0;
        lo[j] = std::min(lo[j], v);
        hi[j] = std::max(hi[j], v);
      }
  const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], 1e-300});
  std::ofstream out(path);
  if (!out) throw fc::IoError("cannot write svg: " + path);
  out << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << w << "\" height=\"" << h
      << "\">\n<rect width=\"100%\" height=\"100%\" fill=\"white\"/>\n";
  const auto dots = [&](const fc::PointSet& ps, const char* color) {
    for (fc::Index i = 0; i < ps.count(); ++i) {
      const double x = ps.pts(i, 0), y = ps.dim() > 1 ? ps.pts(i, 1) : 0.0;
      out << "<circle cx=\"" << pad + (x - lo[0]) / span * (w - 2 * pad) << "\" cy=\""
          << h - pad - (y - lo[1]) / span * (h - 2 * pad) << "\" r=\"1.5\" fill=\"" << color
          << "\"/>\n";
    }
  };
  dots(scene, "#d62728");
  dots(moved, "#1f77b4");
  out << "</svg>\n";
  if (!out) throw fc::IoError("svg write failed: " + path);
}

int cmd_register(const std::vector<std::string>& args) {
  std::vector<std::string> pos;
  fc::RegistrationConfig cfg;
  bool swap = false;
  std::string out_path = "registered.txt", report_path = "report.txt", svg_path;
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    auto value = [&]() -> const std::string& {
      if (i + 1 >= args.size()) throw fc::ParameterError(a + ": missing value");
      return args[++i];
    };
    if (a == "--omega") cfg.omega = to_double(a, value());
    else if (a == "--beta") cfg.beta = to_double(a, value());
    else if (a == "--lambda") cfg.lambda_reg = to_double(a, value());
    else if (a == "--iters") cfg.iterations = static_cast<int>(to_long(a, value()));
    else if (a == "--variant") cfg.variant = fc::variant_from_string(value());
    else if (a == "--rank-fraction") cfg.rank_fraction = to_double(a, value());
    else if (a == "--seed") cfg.seed = static_cast<unsigned long>(to_long(a, value()));
    else if (a == "--no-normalize") cfg.normalize = false;
    else if (a == "--swap") swap = true;
    else if (a == "--early-stop") cfg.early_stop = true;
    else if (a == "--out") out_path = value();
    else if (a == "--report") report_path = value();
    else if (a == "--svg") svg_path = value();
    else if (a == "--device") cfg.device = static_cast<int>(to_long(a, value()));
    else if (!a.empty() && a[0] == '-') throw fc::ParameterError("unknown option: " + a);
    else pos.push_back(a);
  }
  if (pos.size() != 2) throw fc::ParameterError("register: expected MODEL and SCENE files");
  fc::PointSet model = fc::load_points(pos[0]);
  fc::PointSet scene = fc::load_points(pos[1]);
  if (swap) std::swap(model, scene);

  const fc::RegistrationResult res = fc::register_pointsets(model, scene, cfg);
  fc::write_points(res.transformed, out_path);
  fc::write_report(report_path, cfg, res);
  if (!svg_path.empty()) write_overlay_svg(res.transformed, scene, svg_path);

  std::printf("registered %lld points onto %lld in %d iterations\n",
              static_cast<long long>(model.count()), static_cast<long long>(scene.count()),
              static_cast<int>(res.sigma2_trace.size()));
  std::printf("sigma2: %.6g -> %.6g\n", res.sigma2_initial,
              res.sigma2_trace.empty() ? res.sigma2_initial : res.sigma2_trace.back());
  std::printf("t_c=%.6f t_eig=%.6f t_iter=%.6f t_total=%.6f t_setup=%.6f\n", res.timing.t_c,
              res.timing.t_eig, res.timing.t_iter, res.timing.t_total, res.timing.t_setup);
  return 0;
}

// `fcpd bench` (proj/tools/fcpd.cpp:132-182): one registration per
// (size, variant) cell through run_benchmark, written in the reference's CSV
// schema.  --synthetic draws the reference's torus-like cloud.
int cmd_bench(const std::vector<std::string>& args) {
  std::vector<std::string> pos;
  fc::RegistrationConfig cfg;
  std::string sizes_arg, variants_arg = "fast,fast-lowrank", csv_path = "bench.csv",
              svg_path = "bench.svg";
  bool synthetic = false;
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    auto value = [&]() -> const std::string& {
      if (i + 1 >= args.size()) throw fc::ParameterError(a + ": missing value");
      return args[++i];
    };
    if (a == "--sizes") sizes_arg = value();
    else if (a == "--variants") variants_arg = value();
    else if (a == "--iters") cfg.iterations = static_cast<int>(to_long(a, value()));
    else if (a == "--seed") cfg.seed = static_cast<unsigned long>(to_long(a, value()));
    else if (a == "--omega") cfg.omega = to_double(a, value());
    else if (a == "--beta") cfg.beta = to_double(a, value());
    else if (a == "--lambda") cfg.lambda_reg = to_double(a, value());
    else if (a == "--rank-fraction") cfg.rank_fraction = to_double(a, value());
    else if (a == "--csv") csv_path = value();
    else if (a == "--svg") svg_path = value();
    else if (a == "--synthetic") synthetic = true;
    else if (a == "--device") cfg.device = static_cast<int>(to_long(a, value()));
    else if (!a.empty() && a[0] == '-') throw fc::ParameterError("unknown option: " + a);
    else pos.push_back(a);
  }
  std::vector<fc::Index> sizes;
  std::vector<fc::SolverVariant> variants;
  {
    std::stringstream ss(sizes_arg);
    std::string tok;
    while (std::getline(ss, tok, ',')) sizes.push_back(static_cast<fc::Index>(to_long("--sizes", tok)));
    std::stringstream vs(variants_arg);
    while (std::getline(vs, tok, ',')) variants.push_back(fc::variant_from_string(tok));
  }
  if (sizes.empty() || variants.empty())
    throw fc::ParameterError("bench: --sizes and --variants must be non-empty");
  fc::PointSet source;
  if (synthetic) {  // torus-like 3-D cloud with enough points for the largest cell
    const fc::Index m = *std::max_element(sizes.begin(), sizes.end());
    source.pts.resize(m, 3);
    std::mt19937_64 rng(cfg.seed);
    std::uniform_real_distribution<double> u(0.0, 2.0 * 3.14159265358979323846);
    for (fc::Index i = 0; i < m; ++i) {
      const double a = u(rng), b = u(rng);
      source.pts(i, 0) = (1.0 + 0.35 * std::cos(b)) * std::cos(a);
      source.pts(i, 1) = (1.0 + 0.35 * std::cos(b)) * std::sin(a);
      source.pts(i, 2) = 0.35 * std::sin(b);
    }
  } else {
    if (pos.size() != 1) throw fc::ParameterError("bench: expected SOURCE or --synthetic");
    source = fc::load_points(pos[0]);
  }
  const auto records = fc::run_benchmark(source, sizes, variants, cfg, cfg.seed);
  fc::write_bench_csv(records, csv_path);
  fc::write_text_file(fc::bench_plot(records), svg_path);
  for (const auto& r : records)
    std::printf("M=%lld %s t_iter=%.6f t_total=%.6f rmse=%.6g%s\n", static_cast<long long>(r.m),
                fc::to_string(r.variant), r.timing.t_iter, r.timing.t_total, r.rmse,
                r.failed ? " FAILED" : "");
  return 0;
}

// `fcpd plot CSV [--out FILE]` (proj/tools/fcpd.cpp:184-189): re-render a
// bench CSV as the t_iter-vs-M chart.
int cmd_plot(const std::vector<std::string>& args) {
  std::string csv_path, out_path = "plot.svg";
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    if (a == "--out") {
      if (i + 1 >= args.size()) throw fc::ParameterError("--out: missing value");
      out_path = args[++i];
    } else if (!a.empty() && a[0] == '-') {
      throw fc::ParameterError("unknown option: " + a);
    } else if (csv_path.empty()) {
      csv_path = a;
    } else {
      throw fc::ParameterError("plot: expected one CSV file");
    }
  }
  if (csv_path.empty()) throw fc::ParameterError("plot: expected a bench CSV file");
  const auto records = fc::load_bench_csv(csv_path);
  fc::write_text_file(fc::bench_plot(records), out_path);
  std::printf("wrote %s (%zu records)\n", out_path.c_str(), records.size());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(argv[0], 2);
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") return usage(argv[0], 0);
  if (cmd == "--version") {
    std::printf("%s\n", fcpd_version());
    return 0;
  }
  if (cmd != "register" && cmd != "bench" && cmd != "plot") {
    std::fprintf(stderr, "%s: unknown or unsupported subcommand '%s' (this build provides "
                         "'register', 'bench' and 'plot')\n", argv[0], cmd.c_str());
    return 2;
  }
  try {
    const std::vector<std::string> rest(argv + 2, argv + argc);
    if (cmd == "plot") return cmd_plot(rest);
    return cmd == "bench" ? cmd_bench(rest) : cmd_register(rest);
  } catch (const fc::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
