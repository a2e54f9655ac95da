// nlem_denoise_multi_host: whole-image NLEM over a pool of devices (host C++, no device code).
// The image is cut into contiguous row bands, each band runs
// nlem_denoise_rows_host on its device from its own host thread with its own halo of
// S/2 + k/2 rows; no collective runs.  Replaces the reference's internal thread pool
// (NlemParams::threads, proj/src/nlem.cpp:68-90 over proj/include/nlem/parallel.hpp:20-55).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/nlem_b200.h"

namespace {

nlem_status invalid(nlem_failure* f, const char* msg) {
  f->index = -1;
  f->iteration = 0;
  f->kind = 0;
  std::snprintf(f->message, sizeof(f->message), "%s", msg);
  return NLEM_INVALID_ARGUMENT;
}

}  // namespace

extern "C" nlem_status nlem_denoise_multi_host(const float* noisy, int64_t rows, int64_t cols,
                                               const nlem_params* params, float* out,
                                               float* frames, const int32_t* devices,
                                               int32_t ndev, nlem_failure* failure) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  if (rows < 1 || cols < 1) return invalid(f, "image must be non-empty");  // image.hpp:15
  if (nlem_status st = nlem_validate_params(params, f)) return st;
  if (ndev < 1 || devices == nullptr) return invalid(f, "at least one device is required");
  if (!noisy || !out) return invalid(f, "null buffer");
  const int64_t halo = nlem_band_halo(params);
  const int64_t nb = std::min<int64_t>(ndev, rows);
  const int64_t per = (rows + nb - 1) / nb;
  const int64_t T = params->solver_iters;
  std::vector<nlem_failure> fails(nb);
  std::vector<nlem_status> sts(nb, NLEM_OK);
  std::vector<std::vector<float>> band_frames(frames ? nb : 0);
  auto band = [&](int64_t i, int64_t& r0, int64_t& r1) {
    r0 = std::min(rows, i * per);
    r1 = std::min(rows, r0 + per);
  };
  auto run = [&](int64_t i) {
    int64_t r0, r1;
    band(i, r0, r1);
    if (r0 >= r1) return;
    const int64_t i0 = std::max<int64_t>(0, r0 - halo), i1 = std::min(rows, r1 + halo);
    float* fr = nullptr;
    if (frames) {
      band_frames[i].resize(static_cast<size_t>(T) * (r1 - r0) * cols);
      fr = band_frames[i].data();
    }
    sts[i] = nlem_denoise_rows_host(noisy + i0 * cols, i0, i1 - i0, rows, cols, r0, r1 - r0, params,
                                    out + r0 * cols, fr, &fails[i], devices[i]);
  };
  std::vector<std::thread> pool;
  for (int64_t i = 1; i < nb; ++i) pool.emplace_back(run, i);
  run(0);
  for (auto& t : pool) t.join();
  // the first non-numeric error wins; numeric failures report the lowest failing pixel
  int64_t worst = -1;
  for (int64_t i = 0; i < nb; ++i) {
    if (sts[i] == NLEM_OK) continue;
    if (sts[i] != NLEM_NUMERIC_FAILURE) {
      *f = fails[i];
      return sts[i];
    }
    if (worst < 0 || fails[i].index < fails[worst].index) worst = i;
  }
  if (worst >= 0) {
    *f = fails[worst];
    return NLEM_NUMERIC_FAILURE;
  }
  if (frames) {
    for (int64_t i = 0; i < nb; ++i) {
      int64_t r0, r1;
      band(i, r0, r1);
      if (r0 >= r1) continue;
      const size_t bp = static_cast<size_t>(r1 - r0) * cols;
      for (int64_t t = 0; t < T; ++t)
        std::memcpy(frames + (t * rows + r0) * cols, band_frames[i].data() + t * bp,
                    bp * sizeof(float));
    }
  }
  f->index = -1;
  f->iteration = 0;
  f->kind = 0;
  f->message[0] = '\0';
  return NLEM_OK;
}
