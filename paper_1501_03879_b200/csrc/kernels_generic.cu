// Generic (any n, d <= 1024) batched solver kernels and the per-pixel NLEM kernel.
// These are the correctness baseline and the path for shapes the register-tiled
// kernels (kernels_fast.cu) do not specialise.  Persistent grids: each CTA loops
// over problems / pixels.
#include <algorithm>

#include "launch.h"
#include "solver_generic.cuh"

namespace nlemk {

// z = weighted mean of the points.  Default: the reference's points * (w / sum w)
// (types.hpp:71-74, nlem.cpp:17), which stays finite when sum w overflows; with
// `ratio`: sum_k w_k a_k / sum_k w_k, nlm_denoise's form (nlm.cpp:44).  Fixed
// reduction order.  n == 1 gives a_0 exactly (a * (w/w)).
template <int JPL>
__device__ void block_weighted_mean(const float* a, const float* w, int n, int d, GenWork& W,
                                    bool ratio = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (n == 1) {
    for (int j = tid; j < d; j += kGenThreads) W.z[j] = a[j];
    __syncthreads();
    return;
  }
  float den = 0.0f;
  for (int k = warp; k < n; k += kGenWarps) den += w[k];
  if (lane == 0) W.red[warp] = den;
  __syncthreads();
  float D = 0.0f;
#pragma unroll
  for (int i = 0; i < kGenWarps; ++i) D += W.red[i];
  float num[JPL];
#pragma unroll
  for (int q = 0; q < JPL; ++q) num[q] = 0.0f;
  for (int k = warp; k < n; k += kGenWarps) {
    const float* ak = a + static_cast<size_t>(k) * d;
    const float c = ratio ? w[k] : w[k] / D;
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) num[q] = fmaf(ak[j], c, num[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < JPL; ++q) {
    const int j = lane + 32 * q;
    if (j < d) W.gpart[warp * W.dstride + j] = num[q];
  }
  __syncthreads();
  for (int j = tid; j < d; j += kGenThreads) {
    float g = 0.0f;
#pragma unroll
    for (int i = 0; i < kGenWarps; ++i) g += W.gpart[i * W.dstride + j];
    W.z[j] = ratio ? g / D : g;
  }
  __syncthreads();
}

__device__ inline void block_copy(float* dst, const float* src, int64_t count) {
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (vec) {
    const int64_t c4 = count >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int64_t i = threadIdx.x; i < c4; i += blockDim.x) d4[i] = __ldg(s4 + i);
    for (int64_t i = (c4 << 2) + threadIdx.x; i < count; i += blockDim.x) dst[i] = __ldg(src + i);
  } else {
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = __ldg(src + i);
  }
}

template <int JPL, bool SMEM>
__global__ void __launch_bounds__(kGenThreads)
admm_batched_generic(const float* __restrict__ points, const float* __restrict__ weights,
                     int64_t batch, int n, int d, const float* __restrict__ z_init, nlem_box box,
                     float mu, int T, float tol, int res_mode, float* z_out, float* obj_out,
                     int* iters_out, float* tr_obj, float* tr_res, float* scratch,
                     int work_global, FailureSlot* fail, const int* list, const int* list_count,
                     int force_ref) {
  // list: only the listed problems (in list order); force_ref: the reference-form sweep for
  // every problem (collinear point sets, see collinear_kernel)
  extern __shared__ __align__(16) float smem[];
  const size_t nd = static_cast<size_t>(n) * d;
  const size_t ns = admm_state_floats(n, d, force_ref != 0);
  const int64_t count = list ? static_cast<int64_t>(*list_count) : batch;
  // per-CTA global slab (!SMEM): [ns state floats][the work block when it does not fit in
  // shared memory (n beyond ~29k points: the 2n scales and weights)]
  const size_t slab = ns + (work_global ? gen_work_floats(n, d) : 0);
  float* a_s = smem;
  float* p_s = SMEM ? smem + nd : nullptr;
  GenWork W = carve_gen_work(SMEM ? smem + nd + ns
                                  : (work_global ? scratch + blockIdx.x * slab + ns : smem), n, d);
  const int tid = threadIdx.x;
  for (int64_t i = blockIdx.x; i < count; i += gridDim.x) {
    const int64_t b = list ? static_cast<int64_t>(list[i]) : i;
    const float* ag = points + b * nd;
    const float* a;
    float* p;
    if (SMEM) {
      block_copy(a_s, ag, nd);
      a = a_s;
      p = p_s;
    } else {
      a = ag;
      p = scratch + blockIdx.x * slab;
    }
    for (int k = tid; k < n; k += kGenThreads) W.wts[k] = weights[b * n + k];
    __syncthreads();
    if (z_init) {
      for (int j = tid; j < d; j += kGenThreads) W.z[j] = z_init[b * d + j];
      __syncthreads();
    } else {
      block_weighted_mean<JPL>(a, W.wts, n, d, W);  // admm.hpp:40
    }
    const SolveStatus st =
        admm_solve_generic<JPL>(a, W.wts, p, n, d, W, box, mu, T, tol, res_mode,
                                tr_obj ? tr_obj + b * T : nullptr, tr_res ? tr_res + b * T : nullptr,
                                NoSnapshot{}, force_ref != 0);
    __syncthreads();
    if (st.fail_iter >= 0) {
      if (tid == 0) record_failure(fail, b, st.fail_iter, st.fail_kind);
      __syncthreads();
      continue;
    }
    for (int j = tid; j < d; j += kGenThreads) z_out[b * d + j] = W.z[j];
    if (iters_out && tid == 0) iters_out[b] = st.iterations;
    if (obj_out) {  // admm.hpp:81-84
      const float obj = block_em_cost<JPL>(a, W.wts, n, d, W.z, W.red);
      if (tid == 0) {
        obj_out[b] = obj;
        if (!isfinite(obj)) record_failure(fail, b, st.iterations, NLEM_FAIL_ADMM_OBJECTIVE);
      }
    }
    __syncthreads();
  }
}

template <int JPL, bool SMEM>
__global__ void __launch_bounds__(kGenThreads)
irls_batched_generic(const float* __restrict__ points, const float* __restrict__ weights,
                     int64_t batch, int n, int d, const float* __restrict__ x_init, float eps,
                     int T, float tol, float* x_out, float* obj_out, int* iters_out, float* tr_obj,
                     float* scratch, FailureSlot* fail) {
  extern __shared__ __align__(16) float smem[];
  const size_t nd = static_cast<size_t>(n) * d;
  float* a_s = smem;
  // scratch != null: the work block lives in a per-CTA global slab (too large for shared memory)
  GenWork W = carve_gen_work(SMEM ? smem + nd
                                  : (scratch ? scratch + blockIdx.x * gen_work_floats(n, d) : smem),
                             n, d);
  const int tid = threadIdx.x;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const float* ag = points + b * nd;
    const float* a = ag;
    if (SMEM) {
      block_copy(a_s, ag, nd);
      a = a_s;
    }
    for (int k = tid; k < n; k += kGenThreads) W.wts[k] = weights[b * n + k];
    __syncthreads();
    if (x_init) {
      for (int j = tid; j < d; j += kGenThreads) W.z[j] = x_init[b * d + j];
      __syncthreads();
    } else {
      block_weighted_mean<JPL>(a, W.wts, n, d, W);  // irls.hpp:32
    }
    const SolveStatus st = irls_solve_generic<JPL>(a, W.wts, n, d, W, eps, T, tol,
                                                   tr_obj ? tr_obj + b * T : nullptr, NoSnapshot{});
    __syncthreads();
    if (st.fail_iter >= 0) {
      if (tid == 0) record_failure(fail, b, st.fail_iter, st.fail_kind);
      __syncthreads();
      continue;
    }
    for (int j = tid; j < d; j += kGenThreads) x_out[b * d + j] = W.z[j];
    if (iters_out && tid == 0) iters_out[b] = st.iterations;
    if (obj_out) {
      const float obj = block_em_cost<JPL>(a, W.wts, n, d, W.z, W.red);
      if (tid == 0) {
        obj_out[b] = obj;
        if (!isfinite(obj)) record_failure(fail, b, st.iterations, NLEM_FAIL_IRLS_OBJECTIVE);
      }
    }
    __syncthreads();
  }
}

// proj/src/patch.cpp:9-16
__device__ __forceinline__ int64_t mirror_index_dev(int64_t i, int64_t n) {
  if (n == 1) return 0;
  const int64_t period = 2 * (n - 1);
  int64_t m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - m;
}

// Mirror-padded band: pad[pr][pc] = image(mirror(pad_row0 + pr), mirror(pc - col_off)).
// TMA has no mirror mode, so padding once keeps every later patch read in bounds.
// Rows outside the caller's band (only possible when a kernel's fixed tile border exceeds the
// window's S/2 + k/2, i.e. a masked window smaller than the kernel's grid) are clamped to the
// band: they are read by zero-weight grid points only and just have to be finite.
__global__ void pad_band_kernel(const float* __restrict__ in, int64_t in_row0, int64_t in_rows,
                                int64_t rows, int64_t cols, float* __restrict__ pad,
                                int64_t pad_row0, int64_t pad_rows, int64_t pad_cols, int col_off) {
  const int64_t total = pad_rows * pad_cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pr = i / pad_cols, pc = i - pr * pad_cols;
    int64_t gr = mirror_index_dev(pad_row0 + pr, rows);
    gr = gr < in_row0 ? in_row0 : (gr >= in_row0 + in_rows ? in_row0 + in_rows - 1 : gr);
    const int64_t gc = mirror_index_dev(pc - col_off, cols);
    pad[i] = in[(gr - in_row0) * cols + gc];
  }
}

struct FrameSink {  // nlem_denoise_snapshots frames[t-1](r, c) (nlem.cpp:109-125)
  float* frames;
  int64_t plane, pix;
  int center;
  nlem_box box;
  bool clamp;
  __device__ void operator()(int t, const float* z) const {
    if (frames != nullptr && threadIdx.x == 0) {
      const float v = z[center];
      frames[static_cast<int64_t>(t - 1) * plane + pix] = clamp ? clamp_box(v, box) : v;
    }
  }
};

// One CTA per output pixel (persistent loop): gather the clipped window's patches
// (row-major neighbour order, patch.cpp:63-88) from the padded band, Gaussian weights
// (patch.cpp:52-61), init patch (nlem.cpp:13-18), solver (nlem.cpp:20-56), centre
// coordinate out (nlem.cpp:84) and optional per-sweep frames.
template <int JPL, bool SMEM>
__global__ void __launch_bounds__(kGenThreads)
nlem_pixels_generic(const float* __restrict__ pad, int64_t pad_row0, int64_t pad_cols,
                    int64_t rows, int64_t cols, int64_t out_row0, int64_t out_rows, NlemDevParams P,
                    float* out, float* frames, float* scratch, int work_global, FailureSlot* fail) {
  extern __shared__ __align__(16) float smem[];
  const int k = P.patch, hk = k / 2, hs = P.search / 2;
  const int d = k * k;
  const int nmax = P.search * P.search;
  const size_t ndm = static_cast<size_t>(nmax) * d;
  const size_t nsm = static_cast<size_t>(nmax) * d * (d <= kRefFormMaxDim ? 2 : 1);
  // per-CTA global slab (!SMEM): [stack][state][the work block when it does not fit in shared
  // memory (very large search windows)]
  const size_t slab = ndm + nsm + (work_global ? gen_work_floats(nmax, d) : 0);
  float* a_s = SMEM ? smem : scratch + blockIdx.x * slab;
  float* p_s = a_s + ndm;
  GenWork W = carve_gen_work(SMEM ? smem + ndm + nsm : (work_global ? a_s + ndm + nsm : smem), nmax, d);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int center = d / 2;
  const int64_t plane = out_rows * cols;
  for (int64_t pix = blockIdx.x; pix < plane; pix += gridDim.x) {
    const int64_t r = out_row0 + pix / cols, c = pix % cols;
    const int64_t r0 = r - hs > 0 ? r - hs : 0, r1 = r + hs < rows - 1 ? r + hs : rows - 1;
    const int64_t c0 = c - hs > 0 ? c - hs : 0, c1 = c + hs < cols - 1 ? c + hs : cols - 1;
    const int nc = static_cast<int>(c1 - c0 + 1);
    const int n = static_cast<int>((r1 - r0 + 1) * nc);
    const int self = static_cast<int>((r - r0) * nc + (c - c0));
    // gather patches: a[kk][j] = pad(r0 + kk/nc + dr, c0 + kk%nc + dc)
    for (int e = tid; e < n * d; e += kGenThreads) {
      const int kk = e / d, j = e - kk * d;
      const int64_t pr = r0 + kk / nc + (j / k - hk) - pad_row0;
      const int64_t pc = c0 + kk % nc + (j % k - hk) + hs + hk;  // pad col 0 = global -(hs+hk)
      a_s[e] = __ldg(pad + pr * pad_cols + pc);
    }
    __syncthreads();
    // weights exp(-||P_j - P_self||^2 / h^2); the self weight is exactly 1
    for (int kk = warp; kk < n; kk += kGenWarps) {
      float s2 = 0.0f;
      for (int j = lane; j < d; j += 32) {
        const float t = a_s[kk * d + j] - a_s[self * d + j];
        s2 = fmaf(t, t, s2);
      }
      s2 = warp_sum(s2);
      if (lane == 0) W.wts[kk] = expf(-s2 * P.inv_h2);
    }
    __syncthreads();
    const bool nlm_init = P.solver == NLEM_SOLVER_NLM_ONLY || P.init_mode == NLEM_INIT_NLM_PATCH;
    if (nlm_init) {
      block_weighted_mean<JPL>(a_s, W.wts, n, d, W, P.nlm_ratio != 0);
    } else {
      for (int j = tid; j < d; j += kGenThreads) W.z[j] = a_s[self * d + j];
      __syncthreads();
    }
    const FrameSink sink{frames, plane, pix, center, P.range, P.solver != NLEM_SOLVER_ADMM};
    SolveStatus st{P.iters, -1, 0};
    if (P.solver == NLEM_SOLVER_ADMM) {
      st = admm_solve_generic<JPL>(a_s, W.wts, p_s, n, d, W, P.range, P.mu, P.iters, 0.0f,
                                   RES_EXACT0, nullptr, nullptr, sink);
    } else if (P.solver == NLEM_SOLVER_IRLS) {
      st = irls_solve_generic<JPL>(a_s, W.wts, n, d, W, P.epsilon, P.iters, P.irls_tol, nullptr,
                                   sink);
    } else {
      for (int t = 1; t <= P.iters; ++t) sink(t, W.z);  // nlem.cpp:26-31
    }
    __syncthreads();
    if (tid == 0) {
      if (st.fail_iter >= 0) {
        record_failure(fail, r * cols + c, st.fail_iter, st.fail_kind);
      } else {
        float v = W.z[center];
        if (P.solver != NLEM_SOLVER_ADMM) v = clamp_box(v, P.range);
        out[pix] = v;
        if (frames)  // forward-fill after an early stop (nlem.cpp:109-125)
          for (int t = st.iterations; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pix] = v;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
namespace {

int jpl_for(int d) {
  if (d <= 32) return 1;
  if (d <= 64) return 2;
  if (d <= 128) return 4;
  if (d <= 256) return 8;
  if (d <= 512) return 16;
  return 32;
}

}  // namespace

#define NLEM_DISPATCH_JPL(d, ...)              \
  switch (jpl_for(d)) {                          \
    case 1: { constexpr int J = 1; __VA_ARGS__; break; }  \
    case 2: { constexpr int J = 2; __VA_ARGS__; break; }  \
    case 4: { constexpr int J = 4; __VA_ARGS__; break; }  \
    case 8: { constexpr int J = 8; __VA_ARGS__; break; }  \
    case 16: { constexpr int J = 16; __VA_ARGS__; break; } \
    default: { constexpr int J = 32; __VA_ARGS__; break; } \
  }

cudaError_t launch_admm_generic(const AdmmLaunch& L, cudaStream_t stream, const int* list,
                                const int* list_count, bool force_ref) {
  const DeviceCaps& caps = device_caps();
  const size_t nd = static_cast<size_t>(L.n) * L.d;
  const size_t ns = admm_state_floats(L.n, L.d, force_ref);
  const size_t work = gen_work_floats(L.n, L.d) * sizeof(float);
  const size_t smem_full = (nd + ns) * sizeof(float) + work;
  const bool use_smem = smem_full <= static_cast<size_t>(caps.max_smem_optin);
  // the work block (2n + O(d) floats) itself beyond the opt-in limit: global slab as well
  const bool work_global = !use_smem && work > static_cast<size_t>(caps.max_smem_optin);
  const size_t smem = use_smem ? smem_full : work_global ? 0 : work;
  const int per_sm = use_smem ? std::max<int>(1, static_cast<int>(caps.smem_per_sm / (smem + 1024))) : 2;
  int64_t grid = std::min<int64_t>(L.batch, static_cast<int64_t>(caps.sms) * std::min(per_sm, 8));
  grid = std::max<int64_t>(grid, 1);
  float* scratch = nullptr;
  if (!use_smem) {
    const size_t slab = ns + (work_global ? gen_work_floats(L.n, L.d) : 0);
    cudaError_t e = cudaMallocAsync(&scratch, grid * slab * sizeof(float), stream);
    if (e != cudaSuccess) return e;
  }
  cudaError_t err = cudaSuccess;
  NLEM_DISPATCH_JPL(L.d, {
    if (use_smem) {
      auto kfn = admm_batched_generic<J, true>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.points, L.weights, L.batch, L.n, L.d, L.z_init, L.box, L.mu, L.max_iter, L.tol,
          L.res_mode, L.z_out, L.obj_out, L.iters_out, L.tr_obj, L.tr_res, nullptr, 0, L.fail,
          list, list_count, force_ref ? 1 : 0);
    } else {
      auto kfn = admm_batched_generic<J, false>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.points, L.weights, L.batch, L.n, L.d, L.z_init, L.box, L.mu, L.max_iter, L.tol,
          L.res_mode, L.z_out, L.obj_out, L.iters_out, L.tr_obj, L.tr_res, scratch,
          work_global ? 1 : 0, L.fail, list, list_count, force_ref ? 1 : 0);
    }
  });
  err = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, stream);
  return err;
}

cudaError_t launch_irls_generic(const IrlsLaunch& L, cudaStream_t stream) {
  const DeviceCaps& caps = device_caps();
  const size_t nd = static_cast<size_t>(L.n) * L.d;
  const size_t work = gen_work_floats(L.n, L.d) * sizeof(float);
  const size_t smem_full = nd * sizeof(float) + work;
  const bool use_smem = smem_full <= static_cast<size_t>(caps.max_smem_optin);
  const bool work_global = !use_smem && work > static_cast<size_t>(caps.max_smem_optin);
  const size_t smem = use_smem ? smem_full : work_global ? 0 : work;
  const int per_sm = std::max<int>(1, static_cast<int>(caps.smem_per_sm / (smem + 1024)));
  int64_t grid = std::min<int64_t>(L.batch, static_cast<int64_t>(caps.sms) * std::min(per_sm, 8));
  grid = std::max<int64_t>(grid, 1);
  float* scratch = nullptr;
  if (work_global) {
    cudaError_t e = cudaMallocAsync(&scratch, grid * gen_work_floats(L.n, L.d) * sizeof(float), stream);
    if (e != cudaSuccess) return e;
  }
  NLEM_DISPATCH_JPL(L.d, {
    if (use_smem) {
      auto kfn = irls_batched_generic<J, true>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.points, L.weights, L.batch, L.n, L.d, L.x_init, L.eps, L.max_iter, L.tol, L.x_out,
          L.obj_out, L.iters_out, L.tr_obj, nullptr, L.fail);
    } else {
      auto kfn = irls_batched_generic<J, false>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.points, L.weights, L.batch, L.n, L.d, L.x_init, L.eps, L.max_iter, L.tol, L.x_out,
          L.obj_out, L.iters_out, L.tr_obj, scratch, L.fail);
    }
  });
  cudaError_t err = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, stream);
  return err;
}

cudaError_t launch_pad_band(const float* in, int64_t in_row0, int64_t in_rows, int64_t rows,
                            int64_t cols, float* pad, int64_t pad_row0, int64_t pad_rows,
                            int64_t pad_cols, int hk, cudaStream_t stream) {
  const int64_t total = pad_rows * pad_cols;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads,
                                           static_cast<int64_t>(device_caps().sms) * 16);
  pad_band_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), threads, 0, stream>>>(
      in, in_row0, in_rows, rows, cols, pad, pad_row0, pad_rows, pad_cols, hk);
  return cudaGetLastError();
}

cudaError_t launch_nlem_generic(const NlemLaunch& L, cudaStream_t stream) {
  const DeviceCaps& caps = device_caps();
  const int d = L.P.patch * L.P.patch;
  const int nmax = L.P.search * L.P.search;
  const size_t ndm = static_cast<size_t>(nmax) * d;
  const size_t nsm = static_cast<size_t>(nmax) * d * (d <= kRefFormMaxDim ? 2 : 1);
  const size_t work = gen_work_floats(nmax, d) * sizeof(float);
  const size_t smem_full = (ndm + nsm) * sizeof(float) + work;
  const bool use_smem = smem_full <= static_cast<size_t>(caps.max_smem_optin);
  const bool work_global = !use_smem && work > static_cast<size_t>(caps.max_smem_optin);
  const size_t smem = use_smem ? smem_full : work_global ? 0 : work;
  const int per_sm = std::max<int>(1, static_cast<int>(caps.smem_per_sm / (smem + 1024)));
  const int64_t pixels = L.out_rows * L.cols;
  int64_t grid = std::min<int64_t>(pixels, static_cast<int64_t>(caps.sms) * std::min(per_sm, 8));
  grid = std::max<int64_t>(grid, 1);
  float* scratch = nullptr;
  if (!use_smem) {
    const size_t slab = ndm + nsm + (work_global ? gen_work_floats(nmax, d) : 0);
    cudaError_t e = cudaMallocAsync(&scratch, grid * slab * sizeof(float), stream);
    if (e != cudaSuccess) return e;
  }
  NLEM_DISPATCH_JPL(d, {
    if (use_smem) {
      auto kfn = nlem_pixels_generic<J, true>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.pad, L.pad_row0, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out,
          L.frames, nullptr, 0, L.fail);
    } else {
      auto kfn = nlem_pixels_generic<J, false>;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kfn<<<static_cast<unsigned>(grid), kGenThreads, smem, stream>>>(
          L.pad, L.pad_row0, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out,
          L.frames, scratch, work_global ? 1 : 0, L.fail);
    }
  });
  cudaError_t err = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, stream);
  return err;
}

}  // namespace nlemk
