// Host-side seeded input generation (not on the GPU hot path).
//
//  * nlem_add_gaussian_noise restates the reference library's noise model:
//    GaussianSampler = mt19937_64 + Box-Muller (proj/include/nlem/noise.hpp:15-40),
//    applied in row-major order and NOT clipped (proj/src/noise.cpp:7-17).
//  * nlem_synth_* pin down the BASELINE.json generators exactly as SURVEY.md §8d
//    specifies them (the reference's canonical test images are not available):
//      uniform u = engine() / 2^64 in [0, 1);
//      clean image = ramp 40 + 160 c/(W-1), then `rects` axis-aligned rectangles
//        (top-left floor(u*H), floor(u*W); integer sides 4 + floor(u*(max(4,W/8)-3));
//        intensity 255u), then `disks` (centre (u*H, u*W), radius 2 + u*(max(2,W/16)-2),
//        intensity 255u, pixel (r,c) inside iff (r-cr)^2+(c-cc)^2 <= rad^2),
//        later shapes overwrite earlier ones, clipped to [0,255];
//      noisy = float(clean + sigma * GaussianSampler(noise_seed)), row-major, unclipped;
//      point set b: mt19937_64(seed_base + b); centre c ~ U[50,200]^d; the first
//        n - floor(0.1 n) points ~ N(c, 15^2 I) (Box-Muller on the same engine, the
//        GaussianSampler pairing), the last floor(0.1 n) ~ U[0,255]^d; weights 1 - u.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

#include "../../include/nlem_b200.h"

namespace {

inline double uniform01(std::mt19937_64& eng) {
  return static_cast<double>(eng()) * (1.0 / 18446744073709551616.0);  // / 2^64
}

// proj/include/nlem/noise.hpp:15-40, on a borrowed engine.
struct Gaussian {
  std::mt19937_64& eng;
  double spare = 0.0;
  bool have_spare = false;
  double next() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = (static_cast<double>(eng()) + 1.0) / (static_cast<double>(eng.max()) + 1.0);
    const double u2 = static_cast<double>(eng()) / (static_cast<double>(eng.max()) + 1.0);
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * std::numbers::pi * u2;
    spare = radius * std::sin(angle);
    have_spare = true;
    return radius * std::cos(angle);
  }
};

void clean_image(int64_t H, int64_t W, int32_t rects, int32_t disks, uint64_t seed,
                 std::vector<double>& f) {
  f.assign(static_cast<size_t>(H * W), 0.0);
  for (int64_t r = 0; r < H; ++r)
    for (int64_t c = 0; c < W; ++c)
      f[r * W + c] = W > 1 ? 40.0 + 160.0 * static_cast<double>(c) / static_cast<double>(W - 1) : 40.0;
  std::mt19937_64 eng(seed);
  const int64_t side_max = std::max<int64_t>(4, W / 8);
  for (int32_t i = 0; i < rects; ++i) {
    const int64_t r0 = std::min<int64_t>(H - 1, static_cast<int64_t>(uniform01(eng) * H));
    const int64_t c0 = std::min<int64_t>(W - 1, static_cast<int64_t>(uniform01(eng) * W));
    const int64_t hgt = 4 + static_cast<int64_t>(uniform01(eng) * static_cast<double>(side_max - 3));
    const int64_t wid = 4 + static_cast<int64_t>(uniform01(eng) * static_cast<double>(side_max - 3));
    const double val = 255.0 * uniform01(eng);
    for (int64_t r = r0; r < std::min(H, r0 + hgt); ++r)
      for (int64_t c = c0; c < std::min(W, c0 + wid); ++c) f[r * W + c] = val;
  }
  const double rad_max = std::max<double>(2.0, static_cast<double>(W) / 16.0);
  for (int32_t i = 0; i < disks; ++i) {
    const double cr = uniform01(eng) * static_cast<double>(H);
    const double cc = uniform01(eng) * static_cast<double>(W);
    const double rad = 2.0 + uniform01(eng) * (rad_max - 2.0);
    const double val = 255.0 * uniform01(eng);
    const int64_t ra = std::max<int64_t>(0, static_cast<int64_t>(std::floor(cr - rad)));
    const int64_t rb = std::min<int64_t>(H - 1, static_cast<int64_t>(std::ceil(cr + rad)));
    const int64_t ca = std::max<int64_t>(0, static_cast<int64_t>(std::floor(cc - rad)));
    const int64_t cb = std::min<int64_t>(W - 1, static_cast<int64_t>(std::ceil(cc + rad)));
    for (int64_t r = ra; r <= rb; ++r)
      for (int64_t c = ca; c <= cb; ++c) {
        const double dr = static_cast<double>(r) - cr, dc = static_cast<double>(c) - cc;
        if (dr * dr + dc * dc <= rad * rad) f[r * W + c] = val;
      }
  }
  for (double& v : f) v = std::clamp(v, 0.0, 255.0);
}

}  // namespace

extern "C" {

void nlem_add_gaussian_noise(const double* clean, int64_t count, double sigma, uint64_t seed,
                             double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = clean[i];
  if (sigma == 0.0) return;  // noise.cpp:10
  std::mt19937_64 eng(seed);
  Gaussian g{eng};
  for (int64_t i = 0; i < count; ++i) out[i] += sigma * g.next();
}

void nlem_synth_clean_image(int64_t rows, int64_t cols, int32_t rects, int32_t disks,
                            uint64_t seed, float* clean_out) {
  std::vector<double> f;
  clean_image(rows, cols, rects, disks, seed, f);
  for (size_t i = 0; i < f.size(); ++i) clean_out[i] = static_cast<float>(f[i]);
}

void nlem_synth_noisy_image(int64_t rows, int64_t cols, int32_t rects, int32_t disks, double sigma,
                            uint64_t image_seed, uint64_t noise_seed, float* clean_out,
                            float* noisy_out) {
  std::vector<double> f;
  clean_image(rows, cols, rects, disks, image_seed, f);
  std::vector<double> g(f.size());
  nlem_add_gaussian_noise(f.data(), static_cast<int64_t>(f.size()), sigma, noise_seed, g.data());
  for (size_t i = 0; i < f.size(); ++i) {
    if (clean_out) clean_out[i] = static_cast<float>(f[i]);
    noisy_out[i] = static_cast<float>(g[i]);
  }
}

void nlem_synth_point_sets(int64_t batch, int64_t n, int64_t d, uint64_t seed_base,
                           int64_t first_problem, float* points_out, float* weights_out,
                           int32_t threads) {
  const int64_t n_out = static_cast<int64_t>(0.1 * static_cast<double>(n));
  const int64_t n_in = n - n_out;
  auto one = [&](int64_t i) {
    const int64_t b = first_problem + i;
    std::mt19937_64 eng(seed_base + static_cast<uint64_t>(b));
    std::vector<double> c(static_cast<size_t>(d));
    for (int64_t j = 0; j < d; ++j) c[j] = 50.0 + 150.0 * uniform01(eng);
    float* pts = points_out + i * n * d;
    Gaussian g{eng};
    for (int64_t k = 0; k < n_in; ++k)
      for (int64_t j = 0; j < d; ++j) pts[k * d + j] = static_cast<float>(c[j] + 15.0 * g.next());
    for (int64_t k = n_in; k < n; ++k)
      for (int64_t j = 0; j < d; ++j) pts[k * d + j] = static_cast<float>(255.0 * uniform01(eng));
    for (int64_t k = 0; k < n; ++k) weights_out[i * n + k] = static_cast<float>(1.0 - uniform01(eng));
  };
  unsigned workers = threads > 0 ? static_cast<unsigned>(threads) : std::thread::hardware_concurrency();
  if (workers == 0) workers = 1;
  workers = static_cast<unsigned>(std::min<int64_t>(workers, std::max<int64_t>(1, batch)));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (int64_t i = w; i < batch; i += workers) one(i);
    });
  for (auto& t : pool) t.join();
}

}  // extern "C"
