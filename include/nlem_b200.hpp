// nlem_b200.hpp — header-only C++ host API mirroring the reference library's entry points
// (namespace nlem, proj/include/nlem/{types,admm,irls,nlem}.hpp) on Eigen-free types, with
// every compute call forwarded to the sm_100a C-ABI (nlem_b200.h).  A reference user swaps
//   #include "nlem/admm.hpp"  ->  #include "nlem_b200.hpp"
// and links libnlem_b200.so.  Differences, by design:
//   * Scalar is float (the reference is templated, used with double);
//   * PointSet::points is a std::vector in the reference's d x n column-major order
//     (point k at points[k*d .. k*d+d)), Image is row-major std::vector<float>;
//   * on_iterate callbacks cannot cross the ABI: use nlem_denoise_snapshots / record_trace.
// Errors keep the reference types: std::invalid_argument and nlem::NumericFailure
// (types.hpp:20-31, what() and iteration() as in the reference, pixel-decorated for images).
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "nlem_b200.h"

namespace nlem {

class NumericFailure : public std::runtime_error {
 public:
  NumericFailure(const std::string& what, int64_t iteration)
      : std::runtime_error(what), iteration_(iteration) {}
  int64_t iteration() const { return iteration_; }

 private:
  int64_t iteration_;
};

namespace detail {
inline void raise(nlem_status st, const nlem_failure& f) {
  switch (st) {
    case NLEM_OK: return;
    case NLEM_INVALID_ARGUMENT: throw std::invalid_argument(f.message);
    case NLEM_NUMERIC_FAILURE: throw NumericFailure(f.message, f.iteration);
    default: throw std::runtime_error(f.message[0] ? f.message : "CUDA error");
  }
}
}  // namespace detail

// proj/include/nlem/types.hpp:47-54 (d x n column-major == [n][d] row-major)
struct PointSet {
  std::vector<float> points;
  std::vector<float> weights;
  int64_t d = 0;
  int64_t dim() const { return d; }
  int64_t size() const { return d ? static_cast<int64_t>(points.size()) / d : 0; }
};

// proj/include/nlem/types.hpp:77-107
class BoxConstraint {
 public:
  static BoxConstraint unconstrained() { return BoxConstraint(); }
  static BoxConstraint interval(float lower, float upper) {
    if (!(lower <= upper)) throw std::invalid_argument("box requires lower <= upper");
    BoxConstraint b;
    b.c_.bounded = 1;
    b.c_.lower = lower;
    b.c_.upper = upper;
    return b;
  }
  bool is_bounded() const { return c_.bounded != 0; }
  float lower() const { return is_bounded() ? c_.lower : -std::numeric_limits<float>::infinity(); }
  float upper() const { return is_bounded() ? c_.upper : std::numeric_limits<float>::infinity(); }
  const nlem_box& c() const { return c_; }

 private:
  BoxConstraint() { c_ = nlem_box{0, 0.0f, 0.0f}; }
  nlem_box c_;
};

struct TraceRecord {  // types.hpp:111-117
  int64_t iter = 0;
  float objective = 0.0f;
  float primal_residual = std::numeric_limits<float>::quiet_NaN();
};

struct AdmmConfig {  // types.hpp:119-127
  float mu = 1e-3f;
  int64_t max_iter = 100;
  float tol_primal = 0.0f;
  std::vector<float> z_init;
  bool record_trace = false;
};

struct IrlsConfig {  // types.hpp:129-138
  float epsilon = 1e-6f;
  int64_t max_iter = 100;
  float tol = 0.0f;
  std::vector<float> x_init;
  bool record_trace = false;
};

struct SolverResult {  // types.hpp:143-149
  std::vector<float> minimizer;
  float objective = 0.0f;
  int64_t iterations_run = 0;
  std::vector<TraceRecord> trace;
};

// proj/include/nlem/admm.hpp:26-86, on `device`.
inline SolverResult admm_euclidean_median(const PointSet& ps, const BoxConstraint& box,
                                          const AdmmConfig& cfg, int device = 0) {
  if (ps.weights.size() != static_cast<size_t>(ps.size()))
    throw std::invalid_argument("weight count does not match point count");
  if (!cfg.z_init.empty() && static_cast<int64_t>(cfg.z_init.size()) != ps.dim())
    throw std::invalid_argument("z_init dimension does not match point set");
  const int64_t T = cfg.max_iter;
  SolverResult r;
  r.minimizer.resize(ps.dim());
  int32_t iters = 0;
  std::vector<float> to, tr;
  if (cfg.record_trace && T > 0) {
    to.assign(T, std::numeric_limits<float>::quiet_NaN());
    tr.assign(T, std::numeric_limits<float>::quiet_NaN());
  }
  nlem_admm_config c{cfg.mu, static_cast<int32_t>(T), cfg.tol_primal};
  nlem_failure f;
  detail::raise(nlem_admm_batched_host(ps.points.data(), ps.weights.data(), 1, ps.size(), ps.dim(),
                                       cfg.z_init.empty() ? nullptr : cfg.z_init.data(), box.c(), c,
                                       r.minimizer.data(), &r.objective, &iters,
                                       to.empty() ? nullptr : to.data(),
                                       tr.empty() ? nullptr : tr.data(), &f, device),
                f);
  r.iterations_run = iters;
  for (int64_t t = 0; t < (cfg.record_trace ? iters : 0); ++t) r.trace.push_back({t + 1, to[t], tr[t]});
  return r;
}

// proj/include/nlem/irls.hpp:21-68, on `device`.
inline SolverResult irls_euclidean_median(const PointSet& ps, const IrlsConfig& cfg, int device = 0) {
  if (ps.weights.size() != static_cast<size_t>(ps.size()))
    throw std::invalid_argument("weight count does not match point count");
  if (!cfg.x_init.empty() && static_cast<int64_t>(cfg.x_init.size()) != ps.dim())
    throw std::invalid_argument("x_init dimension does not match point set");
  const int64_t T = cfg.max_iter;
  SolverResult r;
  r.minimizer.resize(ps.dim());
  int32_t iters = 0;
  std::vector<float> to;
  if (cfg.record_trace && T > 0) to.assign(T, std::numeric_limits<float>::quiet_NaN());
  nlem_irls_config c{cfg.epsilon, static_cast<int32_t>(T), cfg.tol};
  nlem_failure f;
  detail::raise(nlem_irls_batched_host(ps.points.data(), ps.weights.data(), 1, ps.size(), ps.dim(),
                                       cfg.x_init.empty() ? nullptr : cfg.x_init.data(), c,
                                       r.minimizer.data(), &r.objective, &iters,
                                       to.empty() ? nullptr : to.data(), &f, device),
                f);
  r.iterations_run = iters;
  for (int64_t t = 0; t < (cfg.record_trace ? iters : 0); ++t)
    r.trace.push_back({t + 1, to[t], std::numeric_limits<float>::quiet_NaN()});
  return r;
}

// proj/include/nlem/image.hpp:12 — row-major grayscale raster
struct Image {
  int64_t rows_ = 0, cols_ = 0;
  std::vector<float> data_;
  Image() = default;
  Image(int64_t r, int64_t c, float v = 0.0f) : rows_(r), cols_(c), data_(r * c, v) {}
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  float& operator()(int64_t r, int64_t c) { return data_[r * cols_ + c]; }
  float operator()(int64_t r, int64_t c) const { return data_[r * cols_ + c]; }
  float* data() { return data_.data(); }
  const float* data() const { return data_.data(); }
};

enum class DenoiseSolver { Admm = NLEM_SOLVER_ADMM, Irls = NLEM_SOLVER_IRLS, NlmOnly = NLEM_SOLVER_NLM_ONLY };
enum class PatchInit { NoisyPatch = NLEM_INIT_NOISY_PATCH, NlmPatch = NLEM_INIT_NLM_PATCH };

struct NlemParams {  // proj/include/nlem/nlem.hpp:23-35 (threads: no GPU meaning)
  int search = 21;
  int patch = 7;
  double h = 0.0;
  double sigma = 0.0;
  DenoiseSolver solver = DenoiseSolver::Admm;
  int solver_iters = 4;
  double mu = 1e-3;
  double epsilon = 1e-6;
  PatchInit init_mode = PatchInit::NoisyPatch;
  BoxConstraint range = BoxConstraint::interval(0.0f, 255.0f);
  unsigned threads = 0;
  double irls_tol = 0.0;  // IrlsConfig::tol for the IRLS solver (reference: 0)

  nlem_params c() const {
    return nlem_params{search, patch, static_cast<float>(h), static_cast<float>(sigma),
                       static_cast<int32_t>(solver), solver_iters, static_cast<float>(mu),
                       static_cast<float>(epsilon), static_cast<int32_t>(init_mode), range.c(),
                       static_cast<float>(irls_tol)};
  }
};

inline PatchInit default_init_mode(double sigma) {  // proj/src/nlm.cpp:13-15
  return static_cast<PatchInit>(nlem_default_init_mode(static_cast<float>(sigma)));
}

inline void validate(const NlemParams& params) {  // proj/src/nlm.cpp:17-29
  const nlem_params p = params.c();
  nlem_failure f;
  detail::raise(nlem_validate_params(&p, &f), f);
}

// proj/src/nlem.cpp:68-90
inline Image nlem_denoise(const Image& noisy, const NlemParams& params, int device = 0) {
  Image out(noisy.rows(), noisy.cols());
  const nlem_params p = params.c();
  nlem_failure f;
  detail::raise(nlem_denoise_host(noisy.data(), noisy.rows(), noisy.cols(), &p, out.data(), nullptr,
                                  &f, device),
                f);
  return out;
}

// proj/src/nlem.cpp:68-90 over a pool of devices (the reference's NlemParams::threads pool,
// parallel.hpp:20-55, becomes one row band per device; bitwise equal to one device)
inline Image nlem_denoise(const Image& noisy, const NlemParams& params,
                          const std::vector<int32_t>& devices) {
  Image out(noisy.rows(), noisy.cols());
  const nlem_params p = params.c();
  nlem_failure f;
  detail::raise(nlem_denoise_multi_host(noisy.data(), noisy.rows(), noisy.cols(), &p, out.data(),
                                        nullptr, devices.data(),
                                        static_cast<int32_t>(devices.size()), &f),
                f);
  return out;
}

// proj/src/nlem.cpp:92-128
inline std::vector<Image> nlem_denoise_snapshots(const Image& noisy, const NlemParams& params,
                                                 int device = 0) {
  const nlem_params p = params.c();
  Image out(noisy.rows(), noisy.cols());
  std::vector<float> frames(static_cast<size_t>(params.solver_iters > 0 ? params.solver_iters : 0) *
                            noisy.rows() * noisy.cols());
  nlem_failure f;
  detail::raise(nlem_denoise_host(noisy.data(), noisy.rows(), noisy.cols(), &p, out.data(),
                                  frames.data(), &f, device),
                f);
  std::vector<Image> res;
  const size_t plane = static_cast<size_t>(noisy.rows() * noisy.cols());
  for (int t = 0; t < params.solver_iters; ++t) {
    Image im(noisy.rows(), noisy.cols());
    std::copy(frames.begin() + t * plane, frames.begin() + (t + 1) * plane, im.data_.begin());
    res.push_back(std::move(im));
  }
  return res;
}

// proj/src/patch.cpp:9-16: whole-sample reflection (..., 2, 1, 0, 1, 2, ...), period 2 (n - 1)
inline int64_t mirror_index(int64_t i, int64_t n) {
  if (n < 1) throw std::invalid_argument("mirror_index needs a non-empty axis");
  if (n == 1) return 0;
  const int64_t period = 2 * (n - 1);
  const int64_t m = ((i % period) + period) % period;
  return m < n ? m : period - m;
}

// proj/include/nlem/patch.hpp:33-37 (patches d x n column-major == [n][d] row-major)
struct PatchStack {
  std::vector<float> patches;
  std::vector<float> weights;
  int64_t d = 0;
  int64_t self_column = -1;
  int64_t size() const { return d ? static_cast<int64_t>(patches.size()) / d : 0; }
};

// proj/include/nlem/nlem.hpp:52-55
struct PatchSolve {
  std::vector<float> init;
  std::vector<float> patch;
};

// proj/src/patch.cpp:90-114 — one pixel's stack (gathered on `device`)
inline PatchStack build_patch_stack(const Image& image, int64_t row, int64_t col, int search, int k,
                                    double h, int device = 0) {
  PatchStack s;
  s.d = static_cast<int64_t>(k) * k;
  const int64_t cap = static_cast<int64_t>(search > 0 ? search : 0) * (search > 0 ? search : 0);
  s.patches.resize(static_cast<size_t>(cap * s.d));
  s.weights.resize(static_cast<size_t>(cap));
  int64_t n = 0;
  nlem_failure f;
  detail::raise(nlem_patch_stack_host(image.data(), image.rows(), image.cols(), row, col, search, k,
                                      static_cast<float>(h), s.patches.data(), s.weights.data(), &n,
                                      &s.self_column, &f, device),
                f);
  s.patches.resize(static_cast<size_t>(n * s.d));
  s.weights.resize(static_cast<size_t>(n));
  return s;
}

// proj/src/nlem.cpp:13-18 (the self patch, or points * (w / sum w)), computed on `device`
inline std::vector<float> initial_patch(const PatchStack& stack, PatchInit mode, int device = 0);

// proj/include/nlem/nlem.hpp:60-62, proj/src/nlem.cpp:20-56: the initial patch and the solved
// patch (inside params.range) of one stack.  The reference's on_iterate callback cannot cross
// the ABI; nlem_denoise_snapshots gives the per-iteration centre values of whole images.
inline PatchSolve solve_patch(const PatchStack& stack, const NlemParams& params, int device = 0) {
  if (stack.weights.size() != static_cast<size_t>(stack.size()))
    throw std::invalid_argument("weight count does not match point count");
  PatchSolve r;
  r.init.resize(static_cast<size_t>(stack.d));
  r.patch.resize(static_cast<size_t>(stack.d));
  const nlem_params p = params.c();
  nlem_failure f;
  detail::raise(nlem_solve_patch_host(stack.patches.data(), stack.weights.data(), stack.size(),
                                      stack.d, stack.self_column, &p, r.init.data(), r.patch.data(),
                                      &f, device),
                f);
  return r;
}

inline std::vector<float> initial_patch(const PatchStack& stack, PatchInit mode, int device) {
  NlemParams p;  // NlmOnly: no solve beyond the weighted mean; init_mode picks the init
  p.search = p.patch = 1;
  p.h = 1.0;
  p.solver = DenoiseSolver::NlmOnly;
  p.init_mode = mode;
  p.range = BoxConstraint::unconstrained();
  return solve_patch(stack, p, device).init;
}

// proj/src/nlm.cpp:31-51 (host staging through torch-free C-ABI: device path only exists
// as nlm_denoise(device buffers); here stage via the NlmOnly solver of nlem_denoise_host,
// which computes the same centre coordinate of the weighted-mean patch)
inline Image nlm_denoise(const Image& noisy, const NlemParams& params, int device = 0) {
  NlemParams p = params;
  p.solver = DenoiseSolver::NlmOnly;
  return nlem_denoise(noisy, p, device);
}

}  // namespace nlem
