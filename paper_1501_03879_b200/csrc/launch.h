// Internal host-side launch descriptors shared by the C-ABI layer and the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nlem_b200.h"
#include "common.cuh"

namespace nlemk {

struct DeviceCaps {
  int sms = 148;
  int max_smem_optin = 232448;  // per-CTA opt-in limit
  int smem_per_sm = 233472;
  int cc_major = 10, cc_minor = 0;
};

const DeviceCaps& device_caps();  // of the current device (cached per device)

struct AdmmLaunch {
  const float* points;
  const float* weights;
  int64_t batch;
  int n, d;
  const float* z_init;
  nlem_box box;
  float mu;
  int max_iter;
  float tol;
  int res_mode;
  float* z_out;
  float* obj_out;
  int* iters_out;
  float* tr_obj;
  float* tr_res;
  FailureSlot* fail;
  // fused input validation (types.hpp:58-68) in the batched low-rank kernel: lowest
  // (problem << 2 | code), ~0 when valid; nullptr = validated separately or not at all
  unsigned long long* invalid = nullptr;
};

struct IrlsLaunch {
  const float* points;
  const float* weights;
  int64_t batch;
  int n, d;
  const float* x_init;
  float eps;
  int max_iter;
  float tol;
  float* x_out;
  float* obj_out;
  int* iters_out;
  float* tr_obj;
  FailureSlot* fail;
  unsigned long long* invalid = nullptr;  // fused validation in irls_batched_reg (see AdmmLaunch)
};

struct NlemDevParams {
  int search, patch;
  float inv_h2;  // 1 / h^2 (patch.cpp:56)
  int solver, iters;
  float mu, epsilon;
  int init_mode;
  nlem_box range;
  float irls_tol;
  int nlm_ratio;  // nlm_denoise's sum w*a / sum w (nlm.cpp:44) instead of points*(w/sum w)
};

struct NlemLaunch {
  const float* pad;  // mirror-padded band, row 0 = global row pad_row0, col 0 = global col -border
  int64_t pad_row0, pad_rows, pad_cols;
  int64_t rows, cols;          // full image
  int64_t out_row0, out_rows;  // output band
  NlemDevParams P;
  float* out;     // [out_rows][cols]
  float* frames;  // [iters][out_rows][cols] or null
  FailureSlot* fail;
};

// list / list_count (device): only the listed problems; force_ref: reference-form sweep
cudaError_t launch_admm_generic(const AdmmLaunch& L, cudaStream_t stream, const int* list = nullptr,
                                const int* list_count = nullptr, bool force_ref = false);
// Collinear point sets (affine rank 1, not all equal): appends problem indices to list
cudaError_t launch_collinear(const float* points, int64_t batch, int n, int d, int* list,
                             int* count, cudaStream_t stream);
cudaError_t launch_irls_generic(const IrlsLaunch& L, cudaStream_t stream);
cudaError_t launch_pad_band(const float* in, int64_t in_row0, int64_t in_rows, int64_t rows,
                            int64_t cols, float* pad, int64_t pad_row0, int64_t pad_rows,
                            int64_t pad_cols, int col_off, cudaStream_t stream);

cudaError_t launch_nlem_generic(const NlemLaunch& L, cudaStream_t stream);

// Specialised register-tiled kernels (kernels_fast.cu).  Return false when the
// shape is not covered (the caller then uses the generic kernel).
bool admm_fast_supported(const AdmmLaunch& L);
cudaError_t launch_admm_fast(const AdmmLaunch& L, cudaStream_t stream);
// the same kernel over a device-side list of problem indices (count read on the device)
cudaError_t launch_admm_fast_list(const AdmmLaunch& L, const int* list, const int* list_count,
                                  cudaStream_t stream);
// Low-rank (Gram-form) batched kernel for d = 49 (kernels_batched_lr.cu): problems it cannot
// finish exactly (ring overflow, all points equal, non-finite values) are appended to ho_list
// for launch_admm_fast_list.
bool admm_lr_supported(const AdmmLaunch& L);
// probe: NULL or one zeroed int (small-mu probe launch before the main one)
cudaError_t launch_admm_lr(const AdmmLaunch& L, int* ho_list, int* ho_count, int* probe,
                           cudaStream_t stream);
// Register-resident batched IRLS for d = 49 (kernels_batched_lr.cu).
bool irls_reg_supported(const IrlsLaunch& L);
cudaError_t launch_irls_reg(const IrlsLaunch& L, cudaStream_t stream);
// ring length of the low-rank kernel's second build (kernels_nlem_lr_r12.cu): the most sweeps it
// runs in the small-mu regime
constexpr int kLrBigRing = 12;
cudaError_t launch_nlem_lr_ring12(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                                  int* probe, cudaStream_t stream);
bool nlem_tile_supported(const NlemLaunch& L);
int nlem_tile_grid(const NlemLaunch& L);  // grid side (21 or 11) of the tile instantiation for L
cudaError_t launch_nlem_tile(const NlemLaunch& L, cudaStream_t stream);
// tile kernel over a device-side list of band pixel indices (count read on the device)
cudaError_t launch_nlem_tile_list(const NlemLaunch& L, const int* list, const int* list_count,
                                  cudaStream_t stream);
bool nlem_fast_supported(const NlemLaunch& L);
// Low-rank (Gram-form) one-pixel-per-warp kernel (kernels_nlem_lr.cu): pixels whose history
// ring would drop a significant term are appended to ovf_list for the tile kernel.
bool nlem_lr_supported(const NlemLaunch& L);
// probe: NULL, or 2 zeroed ints for the small-mu probe launch (nlem_lr_probe_wanted); when the
// probe predicts the whole band is handed off, *ovf_count becomes -1 (= every pixel)
bool nlem_lr_probe_wanted(const NlemLaunch& L);
cudaError_t launch_nlem_lr(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                           int* probe, cudaStream_t stream);
cudaError_t launch_nlem_fast(const NlemLaunch& L, cudaStream_t stream);

cudaError_t launch_frames_sse(const float* frames, const float* clean, int64_t nframes,
                              int64_t count, double* sse_dev, cudaStream_t stream);
cudaError_t launch_optimality(const float* points, const float* weights, const float* z,
                              int64_t batch, int n, int d, nlem_box box, float* out,
                              cudaStream_t stream);

// validation kernels (types.hpp:58-68, image.hpp:14-17): packed (index << 2 | code), ~0 = ok
cudaError_t launch_validate_points(const float* points, const float* weights, int64_t batch,
                                   int n, int d, unsigned long long* result, cudaStream_t stream);
cudaError_t launch_patch_stack(const float* img, int64_t rows, int64_t cols, int64_t row,
                               int64_t col, int search, int k, float inv_h2, float* patches,
                               float* weights, cudaStream_t stream);
cudaError_t launch_initial_patch(const float* points, const float* weights, int n, int d,
                                 int self_col, int mode, nlem_box box, float* init,
                                 float* mean_box, cudaStream_t stream);
cudaError_t launch_clip(float* x, int d, nlem_box box, cudaStream_t stream);
cudaError_t launch_validate_image(const float* img, int64_t count, unsigned long long* result,
                                  cudaStream_t stream);

}  // namespace nlemk
