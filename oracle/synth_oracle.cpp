// TEST INFRASTRUCTURE — seeded input generators for the oracle side (bench reference arm,
// tests).  An independent restatement of the BASELINE.json input recipes as SURVEY.md §8d
// pins them, so that the reference arm of bench.py builds its inputs without loading the
// product library.  tests/test_synth_independent.py checks that these buffers equal the
// product generator's (paper_1501_03879_b200/csrc/synth.cpp) bit for bit.
//
// Recipe:
//  * uniforms: one mt19937_64 draw scaled by 2^-64;
//  * clean image: ramp 40 + 160 c / (W - 1); then R rectangles (top-left row/col = floor(u H),
//    floor(u W) capped at H-1 / W-1; height and width 4 + floor(u (max(4, W/8) - 3)); value
//    255 u); then D disks (centre (u H, u W), radius 2 + u (max(2, W/16) - 2), value 255 u,
//    filled where dr^2 + dc^2 <= radius^2 over the bounding box); later shapes overwrite;
//    finally clamp to [0, 255];
//  * noise: the reference GaussianSampler (proj/include/nlem/noise.hpp:15-40: Box-Muller on
//    mt19937_64, cosine first, sine cached) added in row-major order, not clipped
//    (proj/src/noise.cpp:7-17); the image is computed in double and stored as float;
//  * point set b: engine seeded with seed_base + b; centre ~ U[50, 200]^d; the first
//    n - floor(0.1 n) points ~ N(centre, 15^2 I) from the Gaussian sampler on the same
//    engine, the rest ~ U[0, 255]^d; weights 1 - u.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <vector>

namespace {

using Engine = std::mt19937_64;

double unit(Engine& e) { return static_cast<double>(e()) / 18446744073709551616.0; }

class BoxMuller {  // noise.hpp:15-40
 public:
  explicit BoxMuller(Engine& e) : e_(e) {}
  double operator()() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    const double scale = static_cast<double>(Engine::max()) + 1.0;
    const double u1 = (static_cast<double>(e_()) + 1.0) / scale;
    const double u2 = static_cast<double>(e_()) / scale;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double phi = 2.0 * std::numbers::pi * u2;
    cache_ = r * std::sin(phi);
    cached_ = true;
    return r * std::cos(phi);
  }

 private:
  Engine& e_;
  double cache_ = 0.0;
  bool cached_ = false;
};

std::vector<double> scene(int64_t H, int64_t W, int32_t R, int32_t D, uint64_t seed) {
  std::vector<double> img(static_cast<size_t>(H * W));
  for (int64_t c = 0; c < W; ++c) {
    const double v = W > 1 ? 40.0 + 160.0 * static_cast<double>(c) / static_cast<double>(W - 1) : 40.0;
    for (int64_t r = 0; r < H; ++r) img[r * W + c] = v;
  }
  Engine e(seed);
  const int64_t side = std::max<int64_t>(4, W / 8) - 3;
  for (int32_t k = 0; k < R; ++k) {
    int64_t top = static_cast<int64_t>(unit(e) * H);
    int64_t left = static_cast<int64_t>(unit(e) * W);
    top = std::min(top, H - 1);
    left = std::min(left, W - 1);
    const int64_t h = 4 + static_cast<int64_t>(unit(e) * static_cast<double>(side));
    const int64_t w = 4 + static_cast<int64_t>(unit(e) * static_cast<double>(side));
    const double v = 255.0 * unit(e);
    const int64_t bottom = std::min(H, top + h), right = std::min(W, left + w);
    for (int64_t r = top; r < bottom; ++r) std::fill(img.begin() + r * W + left, img.begin() + r * W + right, v);
  }
  const double rmax = std::max(2.0, static_cast<double>(W) / 16.0);
  for (int32_t k = 0; k < D; ++k) {
    const double cy = unit(e) * static_cast<double>(H);
    const double cx = unit(e) * static_cast<double>(W);
    const double rad = 2.0 + unit(e) * (rmax - 2.0);
    const double v = 255.0 * unit(e);
    const double rad2 = rad * rad;
    const int64_t r_lo = std::max<int64_t>(0, static_cast<int64_t>(std::floor(cy - rad)));
    const int64_t r_hi = std::min<int64_t>(H - 1, static_cast<int64_t>(std::ceil(cy + rad)));
    const int64_t c_lo = std::max<int64_t>(0, static_cast<int64_t>(std::floor(cx - rad)));
    const int64_t c_hi = std::min<int64_t>(W - 1, static_cast<int64_t>(std::ceil(cx + rad)));
    for (int64_t r = r_lo; r <= r_hi; ++r) {
      const double dy = static_cast<double>(r) - cy;
      for (int64_t c = c_lo; c <= c_hi; ++c) {
        const double dx = static_cast<double>(c) - cx;
        if (dy * dy + dx * dx <= rad2) img[r * W + c] = v;
      }
    }
  }
  for (double& v : img) v = std::min(255.0, std::max(0.0, v));
  return img;
}

}  // namespace

extern "C" {

void oracle_synth_noisy_image(int64_t rows, int64_t cols, int32_t rects, int32_t disks,
                              double sigma, uint64_t image_seed, uint64_t noise_seed,
                              float* clean_out, float* noisy_out) {
  const std::vector<double> img = scene(rows, cols, rects, disks, image_seed);
  Engine e(noise_seed);
  BoxMuller gauss(e);
  for (size_t i = 0; i < img.size(); ++i) {
    double v = img[i];
    if (sigma != 0.0) v += sigma * gauss();  // noise.cpp:10 (sigma 0: unchanged)
    if (clean_out) clean_out[i] = static_cast<float>(img[i]);
    noisy_out[i] = static_cast<float>(v);
  }
}

void oracle_synth_point_sets(int64_t batch, int64_t n, int64_t d, uint64_t seed_base,
                             int64_t first_problem, float* points_out, float* weights_out) {
  const int64_t outliers = static_cast<int64_t>(0.1 * static_cast<double>(n));
  std::vector<double> centre(static_cast<size_t>(d));
  for (int64_t i = 0; i < batch; ++i) {
    Engine e(seed_base + static_cast<uint64_t>(first_problem + i));
    for (auto& c : centre) c = 50.0 + 150.0 * unit(e);
    BoxMuller gauss(e);
    float* p = points_out + i * n * d;
    for (int64_t k = 0; k < n - outliers; ++k)
      for (int64_t j = 0; j < d; ++j) p[k * d + j] = static_cast<float>(centre[j] + 15.0 * gauss());
    for (int64_t k = n - outliers; k < n; ++k)
      for (int64_t j = 0; j < d; ++j) p[k * d + j] = static_cast<float>(255.0 * unit(e));
    for (int64_t k = 0; k < n; ++k) weights_out[i * n + k] = static_cast<float>(1.0 - unit(e));
  }
}

}  // extern "C"
