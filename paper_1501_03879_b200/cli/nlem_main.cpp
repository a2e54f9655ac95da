// nlem — command-line front end on the sm_100a path, mirroring the reference's subcommands,
// options, output grammars and exit codes (proj/tools/nlem_main.cpp):
//   nlem median  <points> [--solver admm|irls] [--iters N] [--mu M] [--eps E] [--range l:u] [--trace CSV]
//   nlem denoise <image.pgm> --out OUT.pgm [--sigma S] [--seed K] [--repeat R] [solver/patch flags]
//   nlem trace   <image.pgm> --trace CSV (--pixel r:c | --psnr) [noise/solver/patch flags]
//   nlem bench   <images...> --sigma S... [--solver M]... [--repeat R] [--seed K] [--out CSV]
// Exit codes: 0 ok, 2 usage / invalid argument / malformed file, 3 numeric failure, 1 other.
// Every solve runs on the GPU through the C-ABI (include/nlem_b200.hpp); the option parser is
// a small hand-written one (the reference's CLI11 is not vendored).
#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "nlem_b200.hpp"
#include "nlem_b200_io.hpp"

namespace {

struct UsageError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct Config {
  std::string input, out, trace_path, solver = "admm", init, range, pixel;
  std::vector<std::string> inputs, methods;
  bool psnr_mode = false;
  double sigma = 0.0;
  std::vector<double> sigmas;
  long long seed = 0;
  int iters = 4;
  double mu = 1e-3, epsilon = 1e-6, h_mult = 10.0;
  int search = 21, patch = 7, repeat = 1;
  unsigned threads = 0;
};

double to_double(const std::string& v, const std::string& flag) {
  std::size_t used = 0;
  double x = 0;
  try {
    x = std::stod(v, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used != v.size() || v.empty()) throw UsageError(flag + ": '" + v + "' is not a number");
  return x;
}

long long to_int(const std::string& v, const std::string& flag) {
  std::size_t used = 0;
  long long x = 0;
  try {
    x = std::stoll(v, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used != v.size() || v.empty()) throw UsageError(flag + ": '" + v + "' is not an integer");
  return x;
}

template <class T>
T positive(T v, const std::string& flag) {
  if (!(v > 0)) throw UsageError(flag + ": value must be positive");
  return v;
}

std::string member(const std::string& v, const std::vector<std::string>& set, const std::string& flag) {
  if (std::find(set.begin(), set.end(), v) == set.end()) {
    std::string all;
    for (const auto& s : set) all += (all.empty() ? "" : ", ") + s;
    throw UsageError(flag + ": '" + v + "' not in {" + all + "}");
  }
  return v;
}

// "a:b" -> (a, b); same grammar and messages as the reference CLI (nlem_main.cpp:57-75):
// exactly one split point with a full number on each side
std::pair<double, double> parse_pair(const std::string& text, const char* flag) {
  const std::string name(flag);
  const std::size_t at = text.find(':');
  const bool shaped = at != std::string::npos && at > 0 && at + 1 < text.size();
  if (!shaped) throw std::invalid_argument(name + " expects the form a:b");
  auto whole_number = [&](const std::string& part) {
    const char* begin = part.c_str();
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(begin, &end);
    const bool ok = end != begin && *end == '\0' && errno != ERANGE;
    if (!ok) throw std::invalid_argument(name + " expects two numbers a:b");
    return v;
  };
  const double lhs = whole_number(text.substr(0, at));
  const double rhs = whole_number(text.substr(at + 1));
  return {lhs, rhs};
}

nlem::BoxConstraint parse_range(const std::string& text, const nlem::BoxConstraint& fallback) {
  if (text.empty()) return fallback;
  const auto [l, u] = parse_pair(text, "--range");
  return nlem::BoxConstraint::interval(static_cast<float>(l), static_cast<float>(u));
}

// Options -> NlemParams (the reference CLI's defaults, nlem_main.cpp:91-108): h scales with
// max(sigma, 1) so it stays positive at sigma 0, the init follows sigma unless --init is given,
// and the result is validated before any work starts.
nlem::NlemParams make_params(const Config& cfg, double sigma, const std::string& solver) {
  static const std::map<std::string, nlem::DenoiseSolver> kSolvers = {
      {"admm", nlem::DenoiseSolver::Admm}, {"irls", nlem::DenoiseSolver::Irls}};
  static const std::map<std::string, nlem::PatchInit> kInits = {
      {"noisy", nlem::PatchInit::NoisyPatch}, {"nlm", nlem::PatchInit::NlmPatch}};
  const auto sv = kSolvers.find(solver);
  const auto in = kInits.find(cfg.init);
  nlem::NlemParams p;
  p.search = cfg.search;
  p.patch = cfg.patch;
  p.sigma = sigma;
  p.h = cfg.h_mult * (sigma > 1.0 ? sigma : 1.0);
  p.solver = sv == kSolvers.end() ? nlem::DenoiseSolver::NlmOnly : sv->second;
  p.solver_iters = cfg.iters;
  p.mu = cfg.mu;
  p.epsilon = cfg.epsilon;
  p.init_mode = in == kInits.end() ? nlem::default_init_mode(sigma) : in->second;
  p.range = parse_range(cfg.range, nlem::BoxConstraint::interval(0.0f, 255.0f));
  p.threads = cfg.threads;
  nlem::validate(p);
  return p;
}

nlem::Image denoise_once(const nlem::Image& noisy, const nlem::NlemParams& p) {
  return p.solver == nlem::DenoiseSolver::NlmOnly ? nlem::nlm_denoise(noisy, p) : nlem::nlem_denoise(noisy, p);
}

std::string fmt(double v) { return nlem::io_detail::g17(v); }

int run_median(const Config& cfg) {  // nlem_main.cpp:116-158
  const nlem::BoxConstraint box = parse_range(cfg.range, nlem::BoxConstraint::unconstrained());
  if (cfg.iters < 1) throw std::invalid_argument("--iters must be at least 1");
  const nlem::PointSet ps = nlem::read_point_set_file(cfg.input);
  nlem::SolverResult res;
  if (cfg.solver == "admm") {
    nlem::AdmmConfig a;
    a.mu = static_cast<float>(cfg.mu);
    a.max_iter = cfg.iters;
    a.record_trace = !cfg.trace_path.empty();
    res = nlem::admm_euclidean_median(ps, box, a);
  } else {
    nlem::IrlsConfig c;
    c.epsilon = static_cast<float>(cfg.epsilon);
    c.max_iter = cfg.iters;
    c.record_trace = !cfg.trace_path.empty();
    res = nlem::irls_euclidean_median(ps, c);
    if (box.is_bounded()) {  // IRLS is unconstrained; impose the box on the final point
      for (auto& v : res.minimizer) v = std::min(std::max(v, box.lower()), box.upper());
      double obj = 0.0;  // em_cost (costs.hpp:13-20), index order
      for (int64_t k = 0; k < ps.size(); ++k) {
        double s = 0.0;
        for (int64_t i = 0; i < ps.dim(); ++i) {
          const double e = static_cast<double>(res.minimizer[i]) - ps.points[k * ps.dim() + i];
          s += e * e;
        }
        obj += ps.weights[k] * std::sqrt(s);
      }
      res.objective = static_cast<float>(obj);
    }
  }
  if (!cfg.trace_path.empty()) nlem::io_detail::save(nlem::encode_trace_csv(res.trace), cfg.trace_path);
  std::string line = "{\"minimizer\":[";
  for (size_t i = 0; i < res.minimizer.size(); ++i) line += (i ? "," : "") + fmt(res.minimizer[i]);
  line += "],\"objective\":" + fmt(res.objective) + ",\"iterations\":" + std::to_string(res.iterations_run) + "}";
  std::printf("%s\n", line.c_str());
  return 0;
}

std::string sibling_path(const std::string& out, const char* tag) {
  const std::filesystem::path p(out);
  std::filesystem::path named = p.parent_path();
  named /= p.stem().string() + tag + p.extension().string();
  return named.string();
}

int run_denoise(const Config& cfg) {  // nlem_main.cpp:169-198
  if (cfg.repeat < 1) throw std::invalid_argument("--repeat must be at least 1");
  if (!(cfg.sigma >= 0.0)) throw std::invalid_argument("--sigma must be nonnegative");
  const nlem::NlemParams params = make_params(cfg, cfg.sigma, cfg.solver);
  const nlem::Image clean = nlem::read_pgm(cfg.input);
  double sn = 0.0, sd = 0.0;
  for (int r = 0; r < cfg.repeat; ++r) {
    const long long seed = cfg.seed + r;
    const nlem::Image noisy = nlem::add_gaussian_noise(clean, cfg.sigma, static_cast<uint64_t>(seed));
    const nlem::Image den = denoise_once(noisy, params);
    const double pn = nlem::psnr(clean, noisy), pd = nlem::psnr(clean, den);
    sn += pn;
    sd += pd;
    std::printf("seed=%lld psnr_noisy=%.6f psnr_denoised=%.6f\n", seed, pn, pd);
    if (r == 0) {
      nlem::write_pgm(noisy, sibling_path(cfg.out, "_noisy"), nlem::PgmFormat::P5);
      nlem::write_pgm(den, cfg.out, nlem::PgmFormat::P5);
    }
  }
  if (cfg.repeat > 1)
    std::printf("mean psnr_noisy=%.6f psnr_denoised=%.6f\n", sn / cfg.repeat, sd / cfg.repeat);
  return 0;
}

int run_trace(const Config& cfg) {  // nlem_main.cpp:202-250
  if (cfg.pixel.empty() == !cfg.psnr_mode)
    throw std::invalid_argument("pick exactly one of --pixel r:c and --psnr");
  if (!(cfg.sigma >= 0.0)) throw std::invalid_argument("--sigma must be nonnegative");
  const nlem::NlemParams params = make_params(cfg, cfg.sigma, cfg.solver);
  const nlem::Image clean = nlem::read_pgm(cfg.input);
  const nlem::Image noisy = nlem::add_gaussian_noise(clean, cfg.sigma, static_cast<uint64_t>(cfg.seed));
  if (cfg.psnr_mode) {
    std::vector<double> q;
    for (const nlem::Image& f : nlem::nlem_denoise_snapshots(noisy, params)) q.push_back(nlem::psnr(clean, f));
    nlem::io_detail::save(nlem::encode_psnr_csv(q), cfg.trace_path);
    return 0;
  }
  if (params.solver == nlem::DenoiseSolver::NlmOnly)
    throw std::invalid_argument("per-pixel traces need --solver admm or irls");
  const auto [rd, cd] = parse_pair(cfg.pixel, "--pixel");
  const auto row = static_cast<int64_t>(rd), col = static_cast<int64_t>(cd);
  if (row != rd || col != cd || row < 0 || row >= noisy.rows() || col < 0 || col >= noisy.cols())
    throw std::invalid_argument("--pixel must name a pixel inside the image");
  const nlem::PatchStack st = nlem::build_patch_stack(noisy, row, col, params.search, params.patch, params.h);
  const std::vector<float> init = nlem::initial_patch(st, params.init_mode);
  nlem::SolverResult res;
  if (params.solver == nlem::DenoiseSolver::Admm) {
    nlem::AdmmConfig a;
    a.mu = static_cast<float>(params.mu);
    a.max_iter = params.solver_iters;
    a.z_init = init;
    a.record_trace = true;
    res = nlem::admm_euclidean_median(nlem::PointSet{st.patches, st.weights, st.d}, params.range, a);
  } else {
    nlem::IrlsConfig c;
    c.epsilon = static_cast<float>(params.epsilon);
    c.max_iter = params.solver_iters;
    c.x_init = init;
    c.record_trace = true;
    res = nlem::irls_euclidean_median(nlem::PointSet{st.patches, st.weights, st.d}, c);
  }
  nlem::io_detail::save(nlem::encode_trace_csv(res.trace), cfg.trace_path);
  return 0;
}

int run_bench(const Config& cfg) {  // nlem_main.cpp:254-303
  if (cfg.repeat < 1) throw std::invalid_argument("--repeat must be at least 1");
  if (cfg.sigmas.empty()) throw std::invalid_argument("--sigma is required");
  for (double s : cfg.sigmas)
    if (!(s >= 0.0)) throw std::invalid_argument("--sigma must be nonnegative");
  const std::vector<std::string> methods = cfg.methods.empty() ? std::vector<std::string>{"admm"} : cfg.methods;
  for (double s : cfg.sigmas)  // validate the whole grid before touching any file
    for (const auto& m : methods) make_params(cfg, s, m);
  std::vector<nlem::BenchRow> rows;
  for (const std::string& path : cfg.inputs) {
    const nlem::Image clean = nlem::read_pgm(path);
    const std::string name = std::filesystem::path(path).stem().string();
    for (double sigma : cfg.sigmas) {
      std::vector<std::vector<double>> ps(methods.size());
      for (int r = 0; r < cfg.repeat; ++r) {
        const nlem::Image noisy = nlem::add_gaussian_noise(clean, sigma, static_cast<uint64_t>(cfg.seed + r));
        for (size_t m = 0; m < methods.size(); ++m)
          ps[m].push_back(nlem::psnr(clean, denoise_once(noisy, make_params(cfg, sigma, methods[m]))));
      }
      for (size_t m = 0; m < methods.size(); ++m) {
        nlem::BenchRow row;
        row.image = name;
        row.sigma = sigma;
        row.method = methods[m];
        row.repeats = cfg.repeat;
        double mean = 0.0;
        for (double v : ps[m]) mean += v;
        mean /= cfg.repeat;
        double var = 0.0;
        if (std::isfinite(mean))
          for (double v : ps[m]) var += (v - mean) * (v - mean);
        row.mean_psnr = mean;
        row.std_psnr = std::sqrt(var / cfg.repeat);
        rows.push_back(row);
      }
    }
  }
  const std::string table = nlem::encode_bench_csv(rows);
  if (cfg.out.empty()) std::fputs(table.c_str(), stdout);
  else nlem::io_detail::save(table, cfg.out);
  return 0;
}

const char* kUsage =
    "Weighted Euclidean medians and non-local patch-based denoising (B200 / sm_100a)\n"
    "usage: nlem {median,denoise,trace,bench} ...\n"
    "  median  POINTS [--solver admm|irls] [--iters N] [--mu M] [--eps E] [--range l:u] [--trace CSV]\n"
    "  denoise IMAGE --out PGM [--sigma S] [--seed K] [--repeat R] [--solver admm|irls|nlm] [--iters N]\n"
    "          [--mu M] [--eps E] [--search S] [--patch K] [--h-mult H] [--init noisy|nlm] [--range l:u]\n"
    "  trace   IMAGE --trace CSV (--pixel r:c | --psnr) [same noise/solver/patch flags]\n"
    "  bench   IMAGES... --sigma S... [--solver M]... [--iters N] [--repeat R] [--seed K] [--out CSV]\n";

// Parses argv into cfg; returns the subcommand.  Option values may be given as "--x v" or
// "--x=v"; --sigma (bench) and positional images take several values.
std::string parse(int argc, char** argv, Config& cfg) {
  if (argc < 2) throw UsageError("a subcommand is required (median, denoise, trace, bench)");
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") return "help";
  member(sub, {"median", "denoise", "trace", "bench"}, "subcommand");
  const bool noise = sub == "denoise" || sub == "trace";
  const bool patchf = sub != "median";
  std::vector<std::string> solvers = sub == "median" ? std::vector<std::string>{"admm", "irls"}
                                                     : std::vector<std::string>{"admm", "irls", "nlm"};
  std::vector<std::string> pos;
  bool out_seen = false, trace_seen = false, sigma_seen = false;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], val;
    bool has_eq = false;
    if (a.rfind("--", 0) == 0) {
      const auto eq = a.find('=');
      if (eq != std::string::npos) {
        val = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_eq = true;
      }
    } else {
      pos.push_back(a);
      continue;
    }
    if (a == "--help" || a == "-h") return "help";
    auto value = [&]() -> std::string {
      if (has_eq) return val;
      if (i + 1 >= argc) throw UsageError(a + " requires a value");
      return argv[++i];
    };
    if (a == "--psnr" && sub == "trace") {
      cfg.psnr_mode = true;
    } else if (a == "--solver") {
      const std::string v = member(value(), solvers, a);
      if (sub == "bench") cfg.methods.push_back(v);
      else cfg.solver = v;
    } else if (a == "--iters") {
      cfg.iters = static_cast<int>(positive(to_int(value(), a), a));
    } else if (a == "--mu") {
      cfg.mu = positive(to_double(value(), a), a);
    } else if (a == "--eps") {
      cfg.epsilon = positive(to_double(value(), a), a);
    } else if (a == "--range") {
      cfg.range = value();
    } else if (a == "--trace" && (sub == "median" || sub == "trace")) {
      cfg.trace_path = value();
      trace_seen = true;
    } else if (a == "--sigma" && (noise || sub == "bench")) {
      sigma_seen = true;
      if (sub == "bench") {
        cfg.sigmas.push_back(to_double(value(), a));
        // further numeric tokens belong to --sigma (a CLI11 vector option)
        while (!has_eq && i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) {
          try {
            cfg.sigmas.push_back(to_double(argv[i + 1], a));
            ++i;
          } catch (const UsageError&) {
            break;
          }
        }
      } else {
        cfg.sigma = to_double(value(), a);
      }
    } else if (a == "--seed" && (noise || sub == "bench")) {
      cfg.seed = to_int(value(), a);
    } else if (a == "--search" && patchf) {
      cfg.search = static_cast<int>(positive(to_int(value(), a), a));
    } else if (a == "--patch" && patchf) {
      cfg.patch = static_cast<int>(positive(to_int(value(), a), a));
    } else if (a == "--h-mult" && patchf) {
      cfg.h_mult = positive(to_double(value(), a), a);
    } else if (a == "--init" && patchf) {
      cfg.init = member(value(), {"noisy", "nlm"}, a);
    } else if (a == "--threads" && patchf) {
      cfg.threads = static_cast<unsigned>(to_int(value(), a));
    } else if (a == "--repeat" && (sub == "denoise" || sub == "bench")) {
      cfg.repeat = static_cast<int>(positive(to_int(value(), a), a));
    } else if (a == "--out" && (sub == "denoise" || sub == "bench")) {
      cfg.out = value();
      out_seen = true;
    } else if (a == "--pixel" && sub == "trace") {
      cfg.pixel = value();
    } else {
      throw UsageError("unknown option " + a + " for '" + sub + "'");
    }
  }
  if (sub == "bench") {
    if (pos.empty()) throw UsageError("images is required");
    if (!sigma_seen) throw UsageError("--sigma is required");
    cfg.inputs = pos;
  } else {
    if (pos.size() != 1) throw UsageError(std::string(sub == "median" ? "points" : "image") +
                                          (pos.empty() ? " is required" : ": too many positional arguments"));
    cfg.input = pos[0];
  }
  if (sub == "denoise" && !out_seen) throw UsageError("--out is required");
  if (sub == "trace" && !trace_seen) throw UsageError("--trace is required");
  return sub;
}

}  // namespace

int main(int argc, char** argv) {
  Config cfg;
  std::string sub;
  try {
    sub = parse(argc, argv, cfg);
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n%s", e.what(), kUsage);
    return 2;
  }
  if (sub == "help") {
    std::fputs(kUsage, stdout);
    return 0;
  }
  try {
    if (sub == "median") return run_median(cfg);
    if (sub == "denoise") return run_denoise(cfg);
    if (sub == "trace") return run_trace(cfg);
    return run_bench(cfg);
  } catch (const nlem::NumericFailure& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const nlem::ParseError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
