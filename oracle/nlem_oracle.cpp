// ============================================================================
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU oracle for the NLEM / EM-ADMM hot path: a plain-C++ (no Eigen), FP64
// restatement of the reference library under /root/reference/proj.  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library, and only as the checker or the CPU
// baseline — never as the thing measured or shipped.
//
// Why a restatement: the reference needs Eigen3 (proj/CMakeLists.txt:12,
// proj/include/nlem/types.hpp:4), which is absent from this image, so it cannot
// be compiled here.  Every function below names the reference
// file:line it follows, keeps FP64, and keeps the reference's index-order
// accumulation so results are thread-count invariant.
// Pinning: tests/test_oracle_kats.py checks this oracle against every inline
// known-answer test the reference's own unit tests hold for this path
// (tests/golden/reference_kats.json, transcribed by tests/golden/make_reference_kats.py).
// Eigen's SIMD reduction order is not reproducible without Eigen, so bitwise
// parity with an Eigen build is unpinned; the KATs pin it at their tolerances.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

using idx = std::int64_t;

// --- errors (proj/include/nlem/types.hpp:20-31) -----------------------------
struct NumericFailure : std::runtime_error {
  NumericFailure(const std::string& what, idx iteration)
      : std::runtime_error(what + " (iteration " + std::to_string(iteration) + ")"),
        iteration_(iteration) {}
  idx iteration_;
};

// --- point set view: points are [n][d] row-major == Eigen d x n col-major ----
struct PointSet {
  const double* points;  // n*d, point k at points + k*d
  const double* weights; // n
  idx n, d;
  const double* col(idx k) const { return points + k * d; }
};

struct Box {
  bool bounded = false;
  double lo = -std::numeric_limits<double>::infinity();
  double hi = std::numeric_limits<double>::infinity();
};

// proj/include/nlem/types.hpp:58-68
void validate(const PointSet& ps) {
  if (ps.n < 1) throw std::invalid_argument("point set must contain at least one point");
  for (idx i = 0; i < ps.n * ps.d; ++i)
    if (!std::isfinite(ps.points[i])) throw std::invalid_argument("point coordinates must be finite");
  bool any_pos = false;
  for (idx k = 0; k < ps.n; ++k) {
    if (!std::isfinite(ps.weights[k]) || ps.weights[k] < 0.0)
      throw std::invalid_argument("weights must be finite and nonnegative");
    any_pos |= ps.weights[k] > 0.0;
  }
  if (!any_pos) throw std::invalid_argument("at least one weight must be positive");
}

static double sum_index_order(const double* v, idx n) {
  double s = 0.0;
  for (idx i = 0; i < n; ++i) s += v[i];
  return s;
}

// proj/include/nlem/types.hpp:71-74 : points * (w / sum w)
void weighted_mean(const PointSet& ps, double* out) {
  const double wsum = sum_index_order(ps.weights, ps.n);
  for (idx j = 0; j < ps.d; ++j) out[j] = 0.0;
  for (idx k = 0; k < ps.n; ++k) {
    const double c = ps.weights[k] / wsum;
    const double* a = ps.col(k);
    for (idx j = 0; j < ps.d; ++j) out[j] += a[j] * c;
  }
}

static double sq_norm_diff(const double* x, const double* y, idx d) {
  double s = 0.0;
  for (idx j = 0; j < d; ++j) {
    const double t = x[j] - y[j];
    s += t * t;
  }
  return s;
}

// proj/include/nlem/costs.hpp:13-20 — index-order accumulation
double em_cost(const PointSet& ps, const double* x) {
  double total = 0.0;
  for (idx k = 0; k < ps.n; ++k) total += ps.weights[k] * std::sqrt(sq_norm_diff(x, ps.col(k), ps.d));
  return total;
}

// proj/include/nlem/costs.hpp:24-33
double surrogate_cost(const PointSet& ps, const double* x, double eps) {
  if (!(eps > 0.0)) throw std::invalid_argument("surrogate epsilon must be positive");
  double total = 0.0;
  for (idx k = 0; k < ps.n; ++k)
    total += ps.weights[k] * std::sqrt(sq_norm_diff(x, ps.col(k), ps.d) + eps);
  return total;
}

// proj/include/nlem/prox.hpp:29-42 — writes the prox into out (may alias v)
void prox_weighted_norm(const double* v, const double* u, idx d, double lambda, double* out) {
  if (!(lambda >= 0.0)) throw std::invalid_argument("pull distance must be nonnegative");
  if (lambda == 0.0) {
    if (out != v) std::memcpy(out, v, sizeof(double) * d);
    return;
  }
  const double dist = std::sqrt(sq_norm_diff(v, u, d));
  if (dist <= lambda) {
    std::memcpy(out, u, sizeof(double) * d);
    return;
  }
  const double f = lambda / dist;
  for (idx j = 0; j < d; ++j) out[j] = v[j] - f * (v[j] - u[j]);
}

// proj/include/nlem/prox.hpp:13-21
void project_ball(const double* y, idx d, double radius, double* out) {
  if (!(radius >= 0.0)) throw std::invalid_argument("ball radius must be nonnegative");
  double s = 0.0;
  for (idx j = 0; j < d; ++j) s += y[j] * y[j];
  const double norm = std::sqrt(s);
  if (norm <= radius) {
    for (idx j = 0; j < d; ++j) out[j] = y[j];
    return;
  }
  for (idx j = 0; j < d; ++j) out[j] = (radius / norm) * y[j];
}

// proj/include/nlem/prox.hpp:45-50
void project_box(double* x, idx d, const Box& box) {
  if (!box.bounded) return;
  for (idx j = 0; j < d; ++j) x[j] = std::min(std::max(x[j], box.lo), box.hi);
}

struct Trace {
  std::vector<double> objective, residual;
};

struct Result {
  std::vector<double> minimizer;
  double objective = 0.0;
  idx iterations = 0;
};

using IterateFn = std::function<void(idx, const double*)>;

// proj/include/nlem/admm.hpp:26-86 (Algorithm 1)
Result admm(const PointSet& ps, const Box& box, double mu, idx max_iter, double tol_primal,
            const double* z_init, Trace* trace, const IterateFn& on_iterate = nullptr) {
  validate(ps);
  if (!(mu > 0.0)) throw std::invalid_argument("penalty mu must be positive");
  if (max_iter < 1) throw std::invalid_argument("max_iter must be at least 1");
  const idx d = ps.d, n = ps.n;
  const double inv_mu = 1.0 / mu;

  std::vector<double> z(d), y(n * d, 0.0), x(n * d), r(d), v(d);
  if (z_init) std::memcpy(z.data(), z_init, sizeof(double) * d);
  else weighted_mean(ps, z.data());

  idx iterations = 0;
  for (idx t = 1; t <= max_iter; ++t) {
    iterations = t;
    std::fill(r.begin(), r.end(), 0.0);
    for (idx k = 0; k < n; ++k) {  // admm.hpp:53-57
      double* yk = &y[k * d];
      double* xk = &x[k * d];
      for (idx j = 0; j < d; ++j) v[j] = z[j] - inv_mu * yk[j];
      prox_weighted_norm(v.data(), ps.col(k), d, inv_mu * ps.weights[k], xk);
      for (idx j = 0; j < d; ++j) r[j] += xk[j] + inv_mu * yk[j];
    }
    for (idx j = 0; j < d; ++j) z[j] = r[j] / double(n);  // admm.hpp:59
    project_box(z.data(), d, box);

    double residual = 0.0;  // admm.hpp:61-65
    for (idx k = 0; k < n; ++k) {
      double* yk = &y[k * d];
      const double* xk = &x[k * d];
      residual = std::max(residual, std::sqrt(sq_norm_diff(xk, z.data(), d)));
      for (idx j = 0; j < d; ++j) yk[j] += mu * (xk[j] - z[j]);
    }
    bool finite = std::isfinite(residual);
    for (idx j = 0; j < d; ++j) finite &= std::isfinite(z[j]);
    if (!finite) throw NumericFailure("non-finite ADMM iterate", t);  // admm.hpp:67-68

    if (trace) {  // admm.hpp:70-74
      const double obj = em_cost(ps, z.data());
      if (!std::isfinite(obj)) throw NumericFailure("non-finite ADMM objective", t);
      trace->objective.push_back(obj);
      trace->residual.push_back(residual);
    }
    if (on_iterate) on_iterate(t, z.data());
    if (residual <= tol_primal) break;  // admm.hpp:77
  }
  Result res;
  res.minimizer = z;
  res.objective = em_cost(ps, z.data());  // admm.hpp:81
  res.iterations = iterations;
  if (!std::isfinite(res.objective)) throw NumericFailure("non-finite ADMM objective", iterations);
  return res;
}

// proj/include/nlem/irls.hpp:21-68
Result irls(const PointSet& ps, double eps, idx max_iter, double tol, const double* x_init,
            Trace* trace, const IterateFn& on_iterate = nullptr) {
  validate(ps);
  if (!(eps > 0.0)) throw std::invalid_argument("epsilon must be positive");
  if (max_iter < 1) throw std::invalid_argument("max_iter must be at least 1");
  const idx d = ps.d, n = ps.n;
  std::vector<double> x(d), beta(n), num(d);
  if (x_init) std::memcpy(x.data(), x_init, sizeof(double) * d);
  else weighted_mean(ps, x.data());

  double previous = surrogate_cost(ps, x.data(), eps);
  if (!std::isfinite(previous)) throw NumericFailure("non-finite IRLS objective", 0);
  idx iterations = 0;
  for (idx t = 1; t <= max_iter; ++t) {
    iterations = t;
    for (idx k = 0; k < n; ++k)
      beta[k] = ps.weights[k] / std::sqrt(sq_norm_diff(x.data(), ps.col(k), d) + eps);
    // x = (points * beta) / beta.sum()   (irls.hpp:48)
    std::fill(num.begin(), num.end(), 0.0);
    for (idx k = 0; k < n; ++k) {
      const double* a = ps.col(k);
      for (idx j = 0; j < d; ++j) num[j] += a[j] * beta[k];
    }
    const double bsum = sum_index_order(beta.data(), n);
    bool finite = true;
    for (idx j = 0; j < d; ++j) {
      x[j] = num[j] / bsum;
      finite &= std::isfinite(x[j]);
    }
    if (!finite) throw NumericFailure("non-finite IRLS iterate", t);
    const double current = surrogate_cost(ps, x.data(), eps);
    if (!std::isfinite(current)) throw NumericFailure("non-finite IRLS objective", t);
    if (trace) {
      trace->objective.push_back(current);
      trace->residual.push_back(std::numeric_limits<double>::quiet_NaN());
    }
    if (on_iterate) on_iterate(t, x.data());
    if (previous - current <= tol * std::abs(previous)) break;  // irls.hpp:58
    previous = current;
  }
  Result res;
  res.minimizer = x;
  res.objective = em_cost(ps, x.data());
  res.iterations = iterations;
  if (!std::isfinite(res.objective)) throw NumericFailure("non-finite IRLS objective", iterations);
  return res;
}

// proj/include/nlem/parallel.hpp:20-55 — atomic work counter, first exception rethrown
void parallel_for(idx count, unsigned threads, const std::function<void(idx)>& fn) {
  unsigned workers = threads != 0 ? threads : std::thread::hardware_concurrency();
  if (workers == 0) workers = 1;
  if (workers == 1 || count <= 1) {
    for (idx i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<idx> next(0);
  std::exception_ptr failure;
  std::mutex failure_mutex;
  auto worker = [&]() {
    for (;;) {
      const idx i = next.fetch_add(1);
      if (i >= count) return;
      try {
        fn(i);
      } catch (...) {
        {
          std::lock_guard<std::mutex> lock(failure_mutex);
          if (!failure) failure = std::current_exception();
        }
        next.store(count);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < workers; ++w) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (failure) std::rethrow_exception(failure);
}

// --- patches (proj/src/patch.cpp) --------------------------------------------
// proj/src/patch.cpp:9-16
idx mirror_index(idx i, idx n) {
  if (n < 1) throw std::invalid_argument("mirror_index needs a non-empty axis");
  if (n == 1) return 0;
  const idx period = 2 * (n - 1);
  idx m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - m;
}

static void check_odd_positive(int v, const char* what) {
  if (v < 1 || v % 2 == 0) throw std::invalid_argument(std::string(what) + " must be odd and positive");
}

struct Image {
  const double* data;
  idx rows, cols;
  double at(idx r, idx c) const { return data[r * cols + c]; }
};

// proj/include/nlem/image.hpp:14-17
void validate_image(const Image& img) {
  if (img.rows < 1 || img.cols < 1) throw std::invalid_argument("image must be non-empty");
  for (idx i = 0; i < img.rows * img.cols; ++i)
    if (!std::isfinite(img.data[i])) throw std::invalid_argument("image intensities must be finite");
}

// proj/src/patch.cpp:27-38 — row-major k x k window, mirrored
void patch_at(const Image& img, idx row, idx col, int k, double* out) {
  check_odd_positive(k, "patch size");
  const idx half = k / 2;
  idx o = 0;
  for (idx dr = -half; dr <= half; ++dr) {
    const idx r = mirror_index(row + dr, img.rows);
    for (idx dc = -half; dc <= half; ++dc) out[o++] = img.at(r, mirror_index(col + dc, img.cols));
  }
}

// proj/src/patch.cpp:40-50
std::vector<double> build_patch_table(const Image& img, int k) {
  validate_image(img);
  check_odd_positive(k, "patch size");
  const idx d = idx(k) * k;
  std::vector<double> table(d * img.rows * img.cols);
  for (idx r = 0; r < img.rows; ++r)
    for (idx c = 0; c < img.cols; ++c) patch_at(img, r, c, k, &table[(r * img.cols + c) * d]);
  return table;
}

// proj/src/patch.cpp:52-61 — exp(-||P_j - P_c||^2 / h^2)
void patch_weights(const double* patches, idx n, idx d, idx center, double h, double* w) {
  if (center < 0 || center >= n) throw std::invalid_argument("patch_weights center column out of range");
  if (!(h > 0.0)) throw std::invalid_argument("similarity bandwidth h must be positive");
  const double inv_h2 = 1.0 / (h * h);
  for (idx j = 0; j < n; ++j)
    w[j] = std::exp(-sq_norm_diff(patches + j * d, patches + center * d, d) * inv_h2);
}

struct PatchStack {
  std::vector<double> patches;  // n x d (point-contiguous)
  std::vector<double> weights;
  idx n = 0, d = 0, self_column = -1;
};

// proj/src/patch.cpp:63-88 — clipped window, row-major neighbour order
// table_row0: first image row held by `table` (a band of the full table).
PatchStack build_patch_stack(const std::vector<double>& table, idx rows, idx cols, idx row,
                             idx col, int search, int k, double h, idx table_row0 = 0) {
  check_odd_positive(search, "search window");
  if (row < 0 || row >= rows || col < 0 || col >= cols) throw std::invalid_argument("pixel outside the image");
  const idx d = idx(k) * k;
  const idx half = search / 2;
  const idx r0 = std::max<idx>(0, row - half), r1 = std::min<idx>(rows - 1, row + half);
  const idx c0 = std::max<idx>(0, col - half), c1 = std::min<idx>(cols - 1, col + half);
  PatchStack s;
  s.d = d;
  s.n = (r1 - r0 + 1) * (c1 - c0 + 1);
  s.patches.resize(s.n * d);
  idx out = 0;
  for (idx r = r0; r <= r1; ++r)
    for (idx c = c0; c <= c1; ++c) {
      if (r == row && c == col) s.self_column = out;
      std::memcpy(&s.patches[out * d], &table[((r - table_row0) * cols + c) * d], sizeof(double) * d);
      ++out;
    }
  s.weights.resize(s.n);
  patch_weights(s.patches.data(), s.n, d, s.self_column, h, s.weights.data());
  return s;
}

// --- pipeline (proj/src/nlem.cpp, proj/src/nlm.cpp) ---------------------------
enum Solver { ADMM = 0, IRLS = 1, NLM_ONLY = 2 };
enum Init { NOISY_PATCH = 0, NLM_PATCH = 1 };

}  // namespace oracle

extern "C" {

// Plain-C parameter block mirroring nlem::NlemParams (proj/include/nlem/nlem.hpp:23-35),
// plus irls_tol (the reference NLEM path leaves IrlsConfig::tol at 0, irls.hpp:133).
typedef struct {
  int32_t search, patch;
  double h, sigma;
  int32_t solver, solver_iters;
  double mu, epsilon;
  int32_t init_mode;
  int32_t bounded;
  double lo, hi;
  int32_t threads;
  double irls_tol;
} oracle_nlem_params;

typedef struct {
  int64_t index;      // failing problem / pixel (row-major), -1 none
  int64_t iteration;
  char message[256];
} oracle_failure;

}  // extern "C"

namespace oracle {

// proj/src/nlm.cpp:17-29
void validate_params(const oracle_nlem_params& p) {
  if (p.search < 1 || p.search % 2 == 0) throw std::invalid_argument("search window must be odd and positive");
  if (p.patch < 1 || p.patch % 2 == 0) throw std::invalid_argument("patch size must be odd and positive");
  if (p.patch > p.search) throw std::invalid_argument("patch size must not exceed the search window");
  if (!(p.h > 0.0)) throw std::invalid_argument("similarity bandwidth h must be positive");
  if (!(p.sigma >= 0.0)) throw std::invalid_argument("sigma must be nonnegative");
  if (p.solver_iters < 1) throw std::invalid_argument("solver_iters must be at least 1");
  if (!(p.mu > 0.0)) throw std::invalid_argument("penalty mu must be positive");
  if (!(p.epsilon > 0.0)) throw std::invalid_argument("epsilon must be positive");
}

Box box_of(const oracle_nlem_params& p) {
  Box b;
  if (p.bounded) {
    if (!(p.lo <= p.hi)) throw std::invalid_argument("box requires lower <= upper");
    b.bounded = true;
    b.lo = p.lo;
    b.hi = p.hi;
  }
  return b;
}

// proj/src/nlem.cpp:13-18
std::vector<double> initial_patch(const PatchStack& s, int mode) {
  std::vector<double> init(s.d, 0.0);
  if (mode == NOISY_PATCH) {
    std::memcpy(init.data(), &s.patches[s.self_column * s.d], sizeof(double) * s.d);
    return init;
  }
  PointSet ps{s.patches.data(), s.weights.data(), s.n, s.d};
  weighted_mean(ps, init.data());
  return init;
}

// proj/src/nlem.cpp:20-56
std::vector<double> solve_patch(const PatchStack& s, const oracle_nlem_params& p, const Box& box,
                                const IterateFn& on_iterate) {
  std::vector<double> init = initial_patch(s, p.init_mode);
  if (p.solver == NLM_ONLY) {
    std::vector<double> patch = initial_patch(s, NLM_PATCH);
    project_box(patch.data(), s.d, box);
    if (on_iterate)
      for (idx t = 1; t <= p.solver_iters; ++t) on_iterate(t, patch.data());
    return patch;
  }
  PointSet ps{s.patches.data(), s.weights.data(), s.n, s.d};
  if (p.solver == ADMM)
    return admm(ps, box, p.mu, p.solver_iters, 0.0, init.data(), nullptr, on_iterate).minimizer;
  IterateFn cb = nullptr;
  if (on_iterate)
    cb = [&](idx t, const double* x) {
      std::vector<double> c(x, x + s.d);
      project_box(c.data(), s.d, box);
      on_iterate(t, c.data());
    };
  std::vector<double> out =
      irls(ps, p.epsilon, p.solver_iters, p.irls_tol, init.data(), nullptr, cb).minimizer;
  project_box(out.data(), s.d, box);
  return out;
}

}  // namespace oracle

using namespace oracle;

namespace {

int report(const std::exception& e, oracle_failure* f, int64_t index, int64_t iteration) {
  if (f) {
    f->index = index;
    f->iteration = iteration;
    std::snprintf(f->message, sizeof(f->message), "%s", e.what());
  }
  return 0;
}

template <typename Fn>
int guarded(oracle_failure* f, Fn&& fn) {
  if (f) {
    f->index = -1;
    f->iteration = 0;
    f->message[0] = 0;
  }
  try {
    fn();
    return 0;
  } catch (const NumericFailure& e) {
    report(e, f, f ? f->index : -1, e.iteration_);
    return 2;
  } catch (const std::invalid_argument& e) {
    report(e, f, -1, 0);
    return 1;
  } catch (const std::exception& e) {
    report(e, f, -1, 0);
    return 3;
  }
}

// NumericFailure decorated with the pixel (proj/src/nlem.cpp:60-64)
NumericFailure with_pixel(const NumericFailure& e, idx r, idx c) {
  std::string what = e.what();
  // strip the " (iteration N)" suffix the constructor appends, then re-add
  const std::string suffix = " (iteration " + std::to_string(e.iteration_) + ")";
  if (what.size() >= suffix.size() && what.compare(what.size() - suffix.size(), suffix.size(), suffix) == 0)
    what.resize(what.size() - suffix.size());
  return NumericFailure("pixel (" + std::to_string(r) + ", " + std::to_string(c) + "): " + what +
                            suffix,
                        e.iteration_);
}

}  // namespace

extern "C" {

int64_t oracle_mirror_index(int64_t i, int64_t n) {
  try {
    return mirror_index(i, n);
  } catch (...) {
    return -1;
  }
}

int oracle_prox(const double* v, const double* u, int64_t d, double lambda, double* out) {
  return guarded(nullptr, [&] { prox_weighted_norm(v, u, d, lambda, out); });
}

int oracle_project_ball(const double* y, int64_t d, double radius, double* out) {
  return guarded(nullptr, [&] { project_ball(y, d, radius, out); });
}

double oracle_em_cost(const double* pts, const double* w, int64_t n, int64_t d, const double* x) {
  return em_cost(PointSet{pts, w, n, d}, x);
}

double oracle_surrogate_cost(const double* pts, const double* w, int64_t n, int64_t d,
                             const double* x, double eps) {
  try {
    return surrogate_cost(PointSet{pts, w, n, d}, x, eps);
  } catch (...) {
    return std::numeric_limits<double>::quiet_NaN();
  }
}

// Batched proj/include/nlem/admm.hpp:26-86 over B independent problems
// ([B][n][d] points), parallel over problems.  z_init may be NULL (weighted mean).
// trace_* may be NULL, else [B][max_iter] (entries past iterations are left as is).
int oracle_admm_batched(const double* points, const double* weights, int64_t B, int64_t n,
                        int64_t d, const double* z_init, int32_t bounded, double lo, double hi,
                        double mu, int64_t max_iter, double tol_primal, double* z_out,
                        double* objective_out, int64_t* iters_out, double* trace_obj,
                        double* trace_res, int32_t threads, oracle_failure* failure) {
  return guarded(failure, [&] {
    Box box;
    if (bounded) {
      if (!(lo <= hi)) throw std::invalid_argument("box requires lower <= upper");
      box.bounded = true;
      box.lo = lo;
      box.hi = hi;
    }
    if (z_init == nullptr && B > 0 && n >= 1) {
      // z_init empty -> weighted mean (admm.hpp:40)
    }
    std::atomic<int64_t> first_fail(std::numeric_limits<int64_t>::max());
    std::mutex m;
    std::exception_ptr ep;
    parallel_for(B, threads, [&](idx b) {
      PointSet ps{points + b * n * d, weights + b * n, n, d};
      Trace tr;
      try {
        Result r = admm(ps, box, mu, max_iter, tol_primal, z_init ? z_init + b * d : nullptr,
                        (trace_obj || trace_res) ? &tr : nullptr);
        std::memcpy(z_out + b * d, r.minimizer.data(), sizeof(double) * d);
        if (objective_out) objective_out[b] = r.objective;
        if (iters_out) iters_out[b] = r.iterations;
        for (size_t t = 0; t < tr.objective.size(); ++t) {
          if (trace_obj) trace_obj[b * max_iter + t] = tr.objective[t];
          if (trace_res) trace_res[b * max_iter + t] = tr.residual[t];
        }
      } catch (const NumericFailure& e) {
        std::lock_guard<std::mutex> lock(m);
        if (b < first_fail.load()) {  // lowest failing problem, deterministic
          first_fail.store(b);
          ep = std::current_exception();
        }
      }
    });
    if (ep) {
      if (failure) failure->index = first_fail.load();
      std::rethrow_exception(ep);
    }
  });
}

int oracle_irls_batched(const double* points, const double* weights, int64_t B, int64_t n,
                        int64_t d, const double* x_init, double eps, int64_t max_iter, double tol,
                        double* x_out, double* objective_out, int64_t* iters_out,
                        double* trace_obj, int32_t threads, oracle_failure* failure) {
  return guarded(failure, [&] {
    std::atomic<int64_t> first_fail(std::numeric_limits<int64_t>::max());
    std::mutex m;
    std::exception_ptr ep;
    parallel_for(B, threads, [&](idx b) {
      PointSet ps{points + b * n * d, weights + b * n, n, d};
      Trace tr;
      try {
        Result r = irls(ps, eps, max_iter, tol, x_init ? x_init + b * d : nullptr,
                        trace_obj ? &tr : nullptr);
        std::memcpy(x_out + b * d, r.minimizer.data(), sizeof(double) * d);
        if (objective_out) objective_out[b] = r.objective;
        if (iters_out) iters_out[b] = r.iterations;
        for (size_t t = 0; t < tr.objective.size(); ++t) trace_obj[b * max_iter + t] = tr.objective[t];
      } catch (const NumericFailure& e) {
        std::lock_guard<std::mutex> lock(m);
        if (b < first_fail.load()) {
          first_fail.store(b);
          ep = std::current_exception();
        }
      }
    });
    if (ep) {
      if (failure) failure->index = first_fail.load();
      std::rethrow_exception(ep);
    }
  });
}

// proj/src/patch.cpp:90-114 — image-backed stack (patches [n][d], weights [n]).
// Buffers must hold search^2 * patch^2 / search^2 entries; returns n via n_out.
int oracle_build_patch_stack(const double* img, int64_t rows, int64_t cols, int64_t row,
                             int64_t col, int32_t search, int32_t k, double h, double* patches,
                             double* weights, int64_t* n_out, int64_t* self_col) {
  return guarded(nullptr, [&] {
    Image im{img, rows, cols};
    validate_image(im);
    check_odd_positive(search, "search window");
    check_odd_positive(k, "patch size");
    std::vector<double> table = build_patch_table(im, k);
    PatchStack s = build_patch_stack(table, rows, cols, row, col, search, k, h);
    std::memcpy(patches, s.patches.data(), sizeof(double) * s.patches.size());
    std::memcpy(weights, s.weights.data(), sizeof(double) * s.weights.size());
    *n_out = s.n;
    *self_col = s.self_column;
  });
}

int oracle_patch_at(const double* img, int64_t rows, int64_t cols, int64_t row, int64_t col,
                    int32_t k, double* out) {
  return guarded(nullptr, [&] { patch_at(Image{img, rows, cols}, row, col, k, out); });
}

// proj/src/patch.cpp:52-61
int oracle_patch_weights(const double* patches, int64_t n, int64_t d, int64_t center, double h,
                         double* w) {
  return guarded(nullptr, [&] { patch_weights(patches, n, d, center, h, w); });
}

// proj/src/nlem.cpp:13-18 over an explicit stack
int oracle_initial_patch(const double* patches, const double* weights, int64_t n, int64_t d,
                         int64_t self_col, int32_t mode, double* out) {
  return guarded(nullptr, [&] {
    PatchStack s;
    s.patches.assign(patches, patches + n * d);
    s.weights.assign(weights, weights + n);
    s.n = n;
    s.d = d;
    s.self_column = self_col;
    std::vector<double> v = initial_patch(s, mode);
    std::memcpy(out, v.data(), sizeof(double) * d);
  });
}

// proj/src/nlem.cpp:68-90 (frames == NULL) and :92-128 (frames = [T][rows][cols]).
// row_begin/row_end restrict the output rows computed (the CPU-baseline sample);
// the stack geometry always uses the full image (global coordinates).
int oracle_nlem_denoise(const double* noisy, int64_t rows, int64_t cols, oracle_nlem_params params,
                        int64_t row_begin, int64_t row_end, double* out, double* frames,
                        oracle_failure* failure) {
  return guarded(failure, [&] {
    Image im{noisy, rows, cols};
    validate_image(im);
    validate_params(params);
    const Box box = box_of(params);
    if (row_begin < 0 || row_end > rows || row_begin > row_end)
      throw std::invalid_argument("row range outside the image");
    const int k = params.patch;
    const idx d = idx(k) * k;
    const idx center = d / 2;
    const int T = params.solver_iters;

    // Patch table restricted to the rows the requested band touches.
    const idx half = params.search / 2;
    const idx t0 = std::max<idx>(0, row_begin - half), t1 = std::min<idx>(rows, row_end + half);
    std::vector<double> table(d * (t1 - t0) * cols);
    for (idx r = t0; r < t1; ++r)
      for (idx c = 0; c < cols; ++c) patch_at(im, r, c, k, &table[((r - t0) * cols + c) * d]);

    std::atomic<int64_t> first_fail(std::numeric_limits<int64_t>::max());
    std::mutex m;
    std::exception_ptr ep;
    const idx count = (row_end - row_begin) * cols;
    parallel_for(count, params.threads, [&](idx i) {
      const idx r = row_begin + i / cols, c = i % cols;
      const idx pix = r * cols + c;
      PatchStack s = build_patch_stack(table, rows, cols, r, c, params.search, k, params.h, t0);
      try {
        if (!frames) {
          out[pix] = solve_patch(s, params, box, nullptr)[center];
          return;
        }
        std::vector<double> values(T);
        idx reached = 0;
        std::vector<double> patch =
            solve_patch(s, params, box, [&](idx t, const double* z) {
              values[t - 1] = z[center];
              reached = t;
            });
        for (idx t = reached; t < T; ++t) values[t] = patch[center];  // forward-fill
        for (int t = 0; t < T; ++t) frames[(idx)t * rows * cols + pix] = values[t];
        out[pix] = patch[center];
      } catch (const NumericFailure& e) {
        std::lock_guard<std::mutex> lock(m);
        if (pix < first_fail.load()) {
          first_fail.store(pix);
          ep = std::make_exception_ptr(with_pixel(e, r, c));
        }
      }
    });
    if (ep) {
      if (failure) failure->index = first_fail.load();
      std::rethrow_exception(ep);
    }
  });
}

// proj/src/nlm.cpp:31-51
int oracle_nlm_denoise(const double* noisy, int64_t rows, int64_t cols, oracle_nlem_params params,
                       double* out) {
  return guarded(nullptr, [&] {
    Image im{noisy, rows, cols};
    validate_image(im);
    validate_params(params);
    const Box box = box_of(params);
    const int k = params.patch;
    const idx d = idx(k) * k, center = d / 2;
    std::vector<double> table = build_patch_table(im, k);
    parallel_for(rows * cols, params.threads, [&](idx pix) {
      const idx r = pix / cols, c = pix % cols;
      PatchStack s = build_patch_stack(table, rows, cols, r, c, params.search, k, params.h);
      double num = 0.0;
      for (idx j = 0; j < s.n; ++j) num += s.weights[j] * s.patches[j * d + center];
      double mean = num / sum_index_order(s.weights.data(), s.n);
      if (box.bounded) mean = std::clamp(mean, box.lo, box.hi);  // nlm.cpp:9-11
      out[pix] = mean;
    });
  });
}

// proj/include/nlem/psnr.hpp:12-24
double oracle_mse(const double* a, const double* b, int64_t count) {
  double s = 0.0;
  for (idx i = 0; i < count; ++i) {
    const double t = a[i] - b[i];
    s += t * t;
  }
  return s / double(count);
}

double oracle_psnr(const double* a, const double* b, int64_t count) {
  const double err = oracle_mse(a, b, count);
  if (err == 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(255.0 * 255.0 / err);
}

// proj/include/nlem/noise.hpp:15-40 + proj/src/noise.cpp:7-17 (unclipped, row-major)
void oracle_add_gaussian_noise(const double* clean, int64_t count, double sigma, uint64_t seed,
                               double* out) {
  std::memcpy(out, clean, sizeof(double) * count);
  if (sigma == 0.0) return;
  std::mt19937_64 eng(seed);
  bool have_spare = false;
  double spare = 0.0;
  for (idx i = 0; i < count; ++i) {
    double g;
    if (have_spare) {
      have_spare = false;
      g = spare;
    } else {
      const double u1 = (static_cast<double>(eng()) + 1.0) / (static_cast<double>(eng.max()) + 1.0);
      const double u2 = static_cast<double>(eng()) / (static_cast<double>(eng.max()) + 1.0);
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * std::numbers::pi * u2;
      spare = radius * std::sin(angle);
      have_spare = true;
      g = radius * std::cos(angle);
    }
    out[i] += sigma * g;
  }
}

// proj/include/nlem/diagnostics.hpp:22-55 — first-order optimality certificate
double oracle_optimality_residual(const double* pts, const double* w, int64_t n, int64_t d,
                                  int32_t bounded, double lo, double hi, const double* z) {
  std::vector<double> g(d, 0.0);
  double ball = 0.0;
  for (idx k = 0; k < n; ++k) {
    const double* a = pts + k * d;
    const double dist = std::sqrt(sq_norm_diff(z, a, d));
    if (dist <= 1e-12) ball += w[k];
    else
      for (idx j = 0; j < d; ++j) g[j] += (w[k] / dist) * (z[j] - a[j]);
  }
  if (bounded)
    for (idx j = 0; j < d; ++j) {
      const bool at_lo = z[j] == lo, at_hi = z[j] == hi;
      if (at_lo && at_hi) g[j] = 0.0;
      else if (at_hi) g[j] = std::max(g[j], 0.0);
      else if (at_lo) g[j] = std::min(g[j], 0.0);
    }
  double s = 0.0;
  for (idx j = 0; j < d; ++j) s += g[j] * g[j];
  return std::max(0.0, std::sqrt(s) - ball);
}

}  // extern "C"
