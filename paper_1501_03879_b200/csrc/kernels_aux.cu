// Auxiliary device reductions next to the hot path:
//  * per-frame squared error -> PSNR for snapshot sweeps (proj/include/nlem/psnr.hpp:12-24),
//    so convergence curves need no T x H x W device-to-host copy;
//  * batched first-order optimality certificate (proj/include/nlem/diagnostics.hpp:22-55),
//    certifying batched EM-ADMM outputs at scale without the CPU oracle;
//  * the single-pixel helpers behind the reference's solve_patch drop-in: the patch stack of
//    one pixel (proj/src/patch.cpp:90-114) and the initial patch (proj/src/nlem.cpp:13-18).
// Both reductions use fixed orders (deterministic).
#include <algorithm>

#include "launch.h"

namespace nlemk {

constexpr int kPsnrThreads = 256;

// partial SSE (double) of frame f over block chunk b -> part[f * nblk + b]
__global__ void __launch_bounds__(kPsnrThreads)
frame_sse_kernel(const float* __restrict__ frames, const float* __restrict__ clean, int64_t count,
                 int nblk, double* part) {
  const int f = blockIdx.y, b = blockIdx.x;
  const float* fr = frames + static_cast<int64_t>(f) * count;
  const int64_t chunk = (count + nblk - 1) / nblk;
  const int64_t i0 = b * chunk, i1 = i0 + chunk < count ? i0 + chunk : count;
  double acc = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kPsnrThreads) {
    const double d = static_cast<double>(fr[i]) - static_cast<double>(clean[i]);
    acc = fma(d, d, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double w[kPsnrThreads / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kPsnrThreads / 32; ++i) t += w[i];
    part[static_cast<int64_t>(f) * nblk + b] = t;
  }
}

__global__ void frame_sse_finish(const double* part, int nblk, int nframes, double* sse) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nframes) return;
  double t = 0.0;
  for (int b = 0; b < nblk; ++b) t += part[static_cast<int64_t>(f) * nblk + b];
  sse[f] = t;
}

cudaError_t launch_frames_sse(const float* frames, const float* clean, int64_t nframes,
                              int64_t count, double* sse_dev, cudaStream_t stream) {
  const int nblk = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(2 * device_caps().sms, (count + kPsnrThreads - 1) / kPsnrThreads)));
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * nblk * nframes, stream);
  if (e != cudaSuccess) return e;
  frame_sse_kernel<<<dim3(nblk, static_cast<unsigned>(nframes)), kPsnrThreads, 0, stream>>>(
      frames, clean, count, nblk, part);
  frame_sse_finish<<<static_cast<unsigned>((nframes + 127) / 128), 128, 0, stream>>>(
      part, nblk, static_cast<int>(nframes), sse_dev);
  e = cudaGetLastError();
  cudaFreeAsync(part, stream);
  return e;
}

// One CTA (256 threads, warp per point) per problem: diagnostics.hpp:22-55 in float with the
// reference's 1e-12 coincidence threshold and active-face absorption.
template <int JPL>
__global__ void __launch_bounds__(256)
optimality_kernel(const float* __restrict__ points, const float* __restrict__ weights,
                  const float* __restrict__ z, int64_t batch, int n, int d, nlem_box box,
                  float* out) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int W = 8;
  float* gpart = sm;             // [W][d]
  float* ball = sm + W * d;      // [W]
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const float* a = points + b * static_cast<int64_t>(n) * d;
    const float* zb = z + b * d;
    float zv[JPL], g[JPL];
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      zv[q] = j < d ? zb[j] : 0.0f;
      g[q] = 0.0f;
    }
    float bl = 0.0f;
    for (int k = warp; k < n; k += W) {
      const float* ak = a + static_cast<int64_t>(k) * d;
      float diff[JPL];
      float s2 = 0.0f;
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        diff[q] = j < d ? zv[q] - ak[j] : 0.0f;
        s2 = fmaf(diff[q], diff[q], s2);
      }
      s2 = warp_sum(s2);
      const float dist = sqrtf(s2);
      const float w = weights[b * n + k];
      if (dist <= 1e-12f) {
        bl += w;
      } else {
        const float f = w / dist;
#pragma unroll
        for (int q = 0; q < JPL; ++q) g[q] = fmaf(f, diff[q], g[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) gpart[warp * d + j] = g[q];
    }
    if (lane == 0) ball[warp] = bl;
    __syncthreads();
    if (warp == 0) {
      float n2 = 0.0f;
      bool inbox = true;
      for (int j = lane; j < d; j += 32) {
        if (box.bounded) inbox &= zb[j] >= box.lower && zb[j] <= box.upper;
        float gj = 0.0f;
        for (int w = 0; w < W; ++w) gj += gpart[w * d + j];
        if (box.bounded) {
          const bool lo = zb[j] == box.lower, hi = zb[j] == box.upper;
          if (lo && hi) gj = 0.0f;
          else if (hi) gj = fmaxf(gj, 0.0f);  // the face absorbs any push upward
          else if (lo) gj = fminf(gj, 0.0f);
        }
        n2 = fmaf(gj, gj, n2);
      }
      n2 = warp_sum(n2);
      if (lane == 0) {
        float bt = 0.0f;
        for (int w = 0; w < W; ++w) bt += ball[w];
        out[b] = fmaxf(0.0f, sqrtf(n2) - bt);
      }
      if (!__all_sync(0xffffffffu, inbox) && lane == 0) {
        out[b] = __int_as_float(0x7fc00000);  // z outside the box: the reference throws
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_optimality(const float* points, const float* weights, const float* z,
                              int64_t batch, int n, int d, nlem_box box, float* out,
                              cudaStream_t stream) {
  const size_t smem = (8 * static_cast<size_t>(d) + 8) * sizeof(float);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(batch, device_caps().sms * 8));
  const int jpl = d <= 32 ? 1 : d <= 64 ? 2 : d <= 128 ? 4 : d <= 256 ? 8 : d <= 512 ? 16 : 32;
  switch (jpl) {
#define NLEM_OPT_CASE(J)                                                                          \
  case J:                                                                                         \
    cudaFuncSetAttribute(optimality_kernel<J>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         static_cast<int>(smem));                                                 \
    optimality_kernel<J><<<static_cast<unsigned>(grid), 256, smem, stream>>>(points, weights, z,  \
                                                                             batch, n, d, box,    \
                                                                             out);                \
    break;
    NLEM_OPT_CASE(1)
    NLEM_OPT_CASE(2)
    NLEM_OPT_CASE(4)
    NLEM_OPT_CASE(8)
    NLEM_OPT_CASE(16)
    NLEM_OPT_CASE(32)
#undef NLEM_OPT_CASE
  }
  return cudaGetLastError();
}

__device__ __forceinline__ int64_t reflect(int64_t i, int64_t n) {  // patch.cpp:9-16
  if (n == 1) return 0;
  const int64_t period = 2 * (n - 1);
  int64_t m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - m;
}

// build_patch_stack(image, row, col, search, k, h) (patch.cpp:90-114) for one pixel, one CTA:
// the clipped window in row-major neighbour order, patch j of k x k mirrored samples
// (patch.cpp:27-38) at patches[j][0..d), weights exp(-||P_j - P_self||^2 / h^2) with the self
// weight exactly 1 (patch.cpp:52-61).
__global__ void __launch_bounds__(256)
patch_stack_kernel(const float* __restrict__ img, int64_t rows, int64_t cols, int64_t row,
                   int64_t col, int search, int k, float inv_h2, float* patches, float* weights) {
  const int64_t hs = search / 2, hk = k / 2, d = static_cast<int64_t>(k) * k;
  const int64_t r0 = row - hs < 0 ? 0 : row - hs, r1 = row + hs > rows - 1 ? rows - 1 : row + hs;
  const int64_t c0 = col - hs < 0 ? 0 : col - hs, c1 = col + hs > cols - 1 ? cols - 1 : col + hs;
  const int64_t nc = c1 - c0 + 1, n = (r1 - r0 + 1) * nc;
  const int64_t self = (row - r0) * nc + (col - c0);
  for (int64_t e = threadIdx.x; e < n * d; e += blockDim.x) {
    const int64_t j = e / d, q = e % d;
    const int64_t r = r0 + j / nc, c = c0 + j % nc;
    const int64_t pr = reflect(r + q / k - hk, rows), pc = reflect(c + q % k - hk, cols);
    patches[e] = img[pr * cols + pc];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j = warp; j < n; j += blockDim.x >> 5) {
    float s = 0.0f;
    for (int64_t q = lane; q < d; q += 32) {
      const float t = patches[j * d + q] - patches[self * d + q];
      s = fmaf(t, t, s);
    }
    s = warp_sum(s);
    if (lane == 0) weights[j] = expf(-s * inv_h2);
  }
}

// initial_patch (nlem.cpp:13-18) of one stack, one CTA: the self column (NoisyPatch) or the
// weighted mean points * (w / sum w) (NlmPatch, types.hpp:73).  `mean_box` (optional) receives
// the weighted mean projected onto `box` - the NlmOnly solve (nlem.cpp:26-31).
__global__ void __launch_bounds__(256)
initial_patch_kernel(const float* __restrict__ points, const float* __restrict__ weights, int n,
                     int d, int self_col, int mode, nlem_box box, float* init, float* mean_box) {
  __shared__ float part[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float s = 0.0f;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += weights[k];
  s = warp_sum(s);
  if (lane == 0) part[warp] = s;
  __syncthreads();
  float wsum = 0.0f;
  for (int w = 0; w < 8; ++w) wsum += part[w];
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float m = 0.0f;
    for (int k = 0; k < n; ++k) m = fmaf(points[static_cast<int64_t>(k) * d + j], weights[k] / wsum, m);
    init[j] = mode == NLEM_INIT_NOISY_PATCH ? points[static_cast<int64_t>(self_col) * d + j] : m;
    if (mean_box) {
      float v = m;
      if (box.bounded) v = v < box.lower ? box.lower : (box.upper < v ? box.upper : v);
      mean_box[j] = v;
    }
  }
}

// project_box (prox.hpp:45-50) of one d-vector in place
__global__ void clip_kernel(float* x, int d, nlem_box box) {
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const float v = x[j];
    if (box.bounded) x[j] = v < box.lower ? box.lower : (box.upper < v ? box.upper : v);
  }
}

// Collinear point sets: a_k = a_0 + t_k e for every k, not all equal (affine rank 1).  Such a
// problem is one-dimensional along e, where the reference's exact-zero residual stop
// (admm.hpp:77 with tol 0) is reachable as in d <= 16 (the reference-form range of the generic
// kernel), so its iteration count is only reproduced by the reference-form sweep.  One CTA per
// problem: e = a_k1 - a_0 for the lowest k1 with a_k1 != a_0, then every u_k = a_k - a_0 must
// satisfy <u_k, e>^2 >= (1 - 1e-9) ||u_k||^2 ||e||^2 (FP64: exact for exactly collinear
// float data).  The second pass re-reads the problem from L1 / L2.
__global__ void __launch_bounds__(256)
collinear_kernel(const float* __restrict__ points, int64_t batch, int n, int d, int* list,
                 int* count) {
  __shared__ int k1;
  __shared__ int all_ok;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nd = static_cast<int64_t>(n) * d;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const float* a = points + b * nd;
    if (threadIdx.x == 0) {
      k1 = n;
      all_ok = 1;
    }
    __syncthreads();
    // pass 1: lowest point differing from a_0 (each thread stops at its first hit: its later
    // elements belong to later points)
    int mine = n;
    for (int64_t e = d + threadIdx.x; e < nd; e += blockDim.x)
      if (a[e] != a[e % d]) {
        mine = static_cast<int>(e / d);
        break;
      }
    mine = __reduce_min_sync(0xffffffffu, mine);
    if (lane == 0 && mine < n) atomicMin(&k1, mine);
    __syncthreads();
    const int kk = k1;
    if (kk < n) {
      const float* ae = a + static_cast<int64_t>(kk) * d;
      double ee = 0.0;
      for (int j = lane; j < d; j += 32) {
        const double u = static_cast<double>(ae[j]) - a[j];
        ee = fma(u, u, ee);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ee += __shfl_xor_sync(0xffffffffu, ee, o);
      // pass 2: every point parallel to e; a warp leaves as soon as any point is not (generic
      // problems fail on their first points)
      for (int k = kk + 1 + warp; k < n; k += 8) {
        if (!*static_cast<volatile int*>(&all_ok)) break;
        const float* ak = a + static_cast<int64_t>(k) * d;
        double ue = 0.0, uu = 0.0;
        for (int j = lane; j < d; j += 32) {
          const double u = static_cast<double>(ak[j]) - a[j];
          const double v = static_cast<double>(ae[j]) - a[j];
          ue = fma(u, v, ue);
          uu = fma(u, u, uu);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ue += __shfl_xor_sync(0xffffffffu, ue, o);
          uu += __shfl_xor_sync(0xffffffffu, uu, o);
        }
        if (!(ue * ue >= (1.0 - 1e-9) * uu * ee)) {
          if (lane == 0) all_ok = 0;  // benign race: every writer stores 0
          break;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && all_ok) list[atomicAdd(count, 1)] = static_cast<int>(b);
    }
    __syncthreads();
  }
}

cudaError_t launch_collinear(const float* points, int64_t batch, int n, int d, int* list,
                             int* count, cudaStream_t stream) {
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(batch, device_caps().sms * 8));
  collinear_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(points, batch, n, d, list,
                                                                     count);
  return cudaGetLastError();
}

cudaError_t launch_patch_stack(const float* img, int64_t rows, int64_t cols, int64_t row,
                               int64_t col, int search, int k, float inv_h2, float* patches,
                               float* weights, cudaStream_t stream) {
  patch_stack_kernel<<<1, 256, 0, stream>>>(img, rows, cols, row, col, search, k, inv_h2, patches,
                                            weights);
  return cudaGetLastError();
}

cudaError_t launch_initial_patch(const float* points, const float* weights, int n, int d,
                                 int self_col, int mode, nlem_box box, float* init,
                                 float* mean_box, cudaStream_t stream) {
  initial_patch_kernel<<<1, 256, 0, stream>>>(points, weights, n, d, self_col, mode, box, init,
                                              mean_box);
  return cudaGetLastError();
}

cudaError_t launch_clip(float* x, int d, nlem_box box, cudaStream_t stream) {
  clip_kernel<<<1, 256, 0, stream>>>(x, d, box);
  return cudaGetLastError();
}

}  // namespace nlemk
