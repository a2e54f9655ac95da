// C-ABI layer (include/nlem_b200.h): host-side validation with the reference's
// messages, buffer management, dispatch to the sm_100a kernels, failure decoding.
// There is no CPU fallback: every compute entry point runs on the GPU or returns
// NLEM_CUDA_ERROR.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "launch.h"
#include "solver_generic.cuh"

namespace nlemk {

namespace {
DeviceCaps query_caps(int dev) {
  DeviceCaps c;
  cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&c.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&c.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&c.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&c.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  // the stream-ordered scratch (padded bands, counters) comes from the device's default pool:
  // keep freed blocks mapped instead of trimming them at every synchronize, so the first call
  // after a host sync does not pay for re-mapping
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return c;
}
}  // namespace

// Fixed per-device storage filled once per device (std::call_once): the returned reference
// stays valid while other host threads (nlem_denoise_multi_host: one per device) query other
// devices for the first time - no container is ever resized.
const DeviceCaps& device_caps() {
  constexpr int kMaxDevices = 64;
  static DeviceCaps caps[kMaxDevices];
  static std::once_flag once[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) {
    thread_local DeviceCaps extra;
    extra = query_caps(dev);
    return extra;
  }
  std::call_once(once[dev], [dev] { caps[dev] = query_caps(dev); });
  return caps[dev];
}

// ---- validation kernels -----------------------------------------------------------
// code 1: non-finite coordinate, 2: weight non-finite or negative, 3: no positive weight
// Weights of each problem (types.hpp:58-68): code 2 for a non-finite or negative weight, 3 when
// no weight is positive; one block per problem.
__global__ void validate_weights_kernel(const float* __restrict__ weights, int64_t batch, int n,
                                        unsigned long long* result) {
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    int bad_w = 0, pos = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const float w = weights[b * n + k];
      bad_w |= !(isfinite(w) && w >= 0.0f);
      pos |= w > 0.0f;
    }
    bad_w = __syncthreads_or(bad_w);
    pos = __syncthreads_or(pos);
    if (threadIdx.x == 0) {
      const int code = bad_w ? 2 : !pos ? 3 : 0;
      if (code) atomicMin(result, (static_cast<unsigned long long>(b) << 2) | code);
    }
  }
}
// Coordinates (code 1): one flat HBM-bound scan of all batch * n * d floats with 16-byte loads
// (four in flight per thread), independent of the problem boundaries; a non-finite element at
// flat index i reports problem i / nd.  atomicMin over (problem << 2 | code) keeps the lowest
// problem and, within it, the reference's check order (coordinates, then weights).
__device__ __forceinline__ void flag_coord(int64_t i, int64_t nd, unsigned long long* result) {
  atomicMin(result, (static_cast<unsigned long long>(i / nd) << 2) | 1ull);
}
__global__ void validate_coords_kernel(const float* __restrict__ points, int64_t total, int64_t nd,
                                       unsigned long long* result) {
  const int64_t lead = static_cast<int64_t>(((16 - (reinterpret_cast<uintptr_t>(points) & 15)) & 15) / 4);
  const int64_t head = lead < total ? lead : total;  // floats before the first 16-byte boundary
  const int64_t nvec = (total - head) / 4;
  const float4* __restrict__ body = reinterpret_cast<const float4*>(points + head);
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (tid < head && !isfinite(points[tid])) flag_coord(tid, nd, result);
  const int64_t tail0 = head + 4 * nvec;
  if (tid < total - tail0 && !isfinite(points[tail0 + tid])) flag_coord(tail0 + tid, nd, result);
  constexpr int U = 4;
  for (int64_t v0 = tid; v0 < nvec; v0 += U * stride) {
    float4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * stride;
      q[u] = v < nvec ? __ldcs(body + v) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float e[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (!isfinite(e[c])) flag_coord(head + 4 * (v0 + u * stride) + c, nd, result);
    }
  }
}

__global__ void validate_image_kernel(const float* __restrict__ img, int64_t count,
                                      unsigned long long* result) {
  int bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(img[i]);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && bad) atomicMin(result, 1ull);
}

cudaError_t launch_validate_points(const float* points, const float* weights, int64_t batch, int n,
                                   int d, unsigned long long* result, cudaStream_t stream) {
  const int64_t nd = static_cast<int64_t>(n) * d, total = batch * nd;
  const int64_t cgrid = std::max<int64_t>(1, std::min<int64_t>((total / 4 + 255) / 256,
                                                                device_caps().sms * 8));
  validate_coords_kernel<<<static_cast<unsigned>(cgrid), 256, 0, stream>>>(points, total, nd, result);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(batch, device_caps().sms * 8));
  validate_weights_kernel<<<static_cast<unsigned>(grid), 128, 0, stream>>>(weights, batch, n, result);
  return cudaGetLastError();
}

cudaError_t launch_validate_image(const float* img, int64_t count, unsigned long long* result,
                                  cudaStream_t stream) {
  const int64_t grid =
      std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, device_caps().sms * 8));
  validate_image_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(img, count, result);
  return cudaGetLastError();
}

}  // namespace nlemk

using namespace nlemk;

namespace {

constexpr int kMaxDim = 1024;

nlem_status invalid(nlem_failure* f, const std::string& msg) {
  if (f) {
    f->index = -1;
    f->iteration = 0;
    f->kind = NLEM_FAIL_NONE;
    std::snprintf(f->message, sizeof(f->message), "%s", msg.c_str());
  }
  return NLEM_INVALID_ARGUMENT;
}

nlem_status cuda_fail(nlem_failure* f, cudaError_t e) {
  if (f) {
    f->index = -1;
    f->iteration = 0;
    f->kind = NLEM_FAIL_NONE;
    std::snprintf(f->message, sizeof(f->message), "CUDA error: %s", cudaGetErrorString(e));
  }
  return NLEM_CUDA_ERROR;
}

void clear(nlem_failure* f) {
  if (f) {
    f->index = -1;
    f->iteration = 0;
    f->kind = NLEM_FAIL_NONE;
    f->message[0] = '\0';
  }
}

const char* kind_text(int kind) {
  switch (kind) {
    case NLEM_FAIL_ADMM_ITERATE: return "non-finite ADMM iterate";
    case NLEM_FAIL_ADMM_OBJECTIVE: return "non-finite ADMM objective";
    case NLEM_FAIL_IRLS_ITERATE: return "non-finite IRLS iterate";
    case NLEM_FAIL_IRLS_OBJECTIVE: return "non-finite IRLS objective";
    default: return "numeric failure";
  }
}

// Decode a FailureSlot; pixel_cols > 0 decorates "pixel (r, c): " (nlem.cpp:60-64).
nlem_status decode_failure(unsigned long long packed, nlem_failure* f, int64_t pixel_cols) {
  if (packed == ~0ull) return NLEM_OK;
  const int64_t index = static_cast<int64_t>(packed >> 24);
  const int64_t iteration = static_cast<int64_t>((packed >> 4) & 0xFFFFF);
  const int kind = static_cast<int>(packed & 0xF);
  if (f) {
    f->index = index;
    f->iteration = iteration;
    f->kind = kind;
    if (pixel_cols > 0)
      std::snprintf(f->message, sizeof(f->message), "pixel (%lld, %lld): %s (iteration %lld)",
                    static_cast<long long>(index / pixel_cols),
                    static_cast<long long>(index % pixel_cols), kind_text(kind),
                    static_cast<long long>(iteration));
    else
      std::snprintf(f->message, sizeof(f->message), "%s (iteration %lld)", kind_text(kind),
                    static_cast<long long>(iteration));
  }
  return NLEM_NUMERIC_FAILURE;
}

struct DevSlot {  // one 8-byte device word for a failure/validation record
  unsigned long long* ptr = nullptr;
  cudaStream_t stream;
  explicit DevSlot(cudaStream_t s) : stream(s) {}
  cudaError_t init() {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ptr), sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(ptr, 0xFF, sizeof(unsigned long long), stream);
  }
  cudaError_t read(unsigned long long* out) {
    cudaError_t e = cudaMemcpyAsync(out, ptr, sizeof(*out), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(stream);
  }
  ~DevSlot() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

nlem_status check_box(const nlem_box& box, nlem_failure* f) {
  if (box.bounded && !(box.lower <= box.upper)) return invalid(f, "box requires lower <= upper");
  return NLEM_OK;
}

nlem_status validate_params_impl(const nlem_params* p, nlem_failure* f) {
  if (p == nullptr) return invalid(f, "params must not be null");
  // proj/src/nlm.cpp:17-29, same order and messages
  if (p->search < 1 || p->search % 2 == 0) return invalid(f, "search window must be odd and positive");
  if (p->patch < 1 || p->patch % 2 == 0) return invalid(f, "patch size must be odd and positive");
  if (p->patch > p->search) return invalid(f, "patch size must not exceed the search window");
  if (!(p->h > 0.0f)) return invalid(f, "similarity bandwidth h must be positive");
  if (!(p->sigma >= 0.0f)) return invalid(f, "sigma must be nonnegative");
  if (p->solver_iters < 1) return invalid(f, "solver_iters must be at least 1");
  if (!(p->mu > 0.0f)) return invalid(f, "penalty mu must be positive");
  if (!(p->epsilon > 0.0f)) return invalid(f, "epsilon must be positive");
  if (p->solver < 0 || p->solver > 2) return invalid(f, "unknown solver");
  if (p->init_mode < 0 || p->init_mode > 1) return invalid(f, "unknown init mode");
  if (p->patch * p->patch > kMaxDim) return invalid(f, "patch dimension k*k above 1024 is not supported");
  return check_box(p->range, f);
}

nlem_status report_invalid(unsigned long long v, nlem_failure* f);
nlem_status validate_points_dev(const float* points, const float* weights, int64_t batch, int n,
                                int d, nlem_failure* f, cudaStream_t s) {
  DevSlot slot(s);
  cudaError_t e = slot.init();
  if (e == cudaSuccess) e = launch_validate_points(points, weights, batch, n, d, slot.ptr, s);
  unsigned long long v = ~0ull;
  if (e == cudaSuccess) e = slot.read(&v);
  if (e != cudaSuccess) return cuda_fail(f, e);
  return report_invalid(v, f);
}

nlem_status report_invalid(unsigned long long v, nlem_failure* f) {
  if (v == ~0ull) return NLEM_OK;
  const int code = static_cast<int>(v & 3);
  // types.hpp:58-68 messages
  const char* msg = code == 1 ? "point coordinates must be finite"
                    : code == 2 ? "weights must be finite and nonnegative"
                                : "at least one weight must be positive";
  nlem_status st = invalid(f, msg);
  if (f) f->index = static_cast<int64_t>(v >> 2);
  return st;
}

int res_mode_for(float tol, bool trace_res) {
  if (trace_res || tol > 0.0f) return RES_FULL;
  if (tol == 0.0f) return RES_EXACT0;
  return RES_NONE;
}

NlemDevParams dev_params(const nlem_params& p) {
  NlemDevParams d;
  d.search = p.search;
  d.patch = p.patch;
  const double h = static_cast<double>(p.h);
  d.inv_h2 = static_cast<float>(1.0 / (h * h));
  d.solver = p.solver;
  d.iters = p.solver_iters;
  d.mu = p.mu;
  d.epsilon = p.epsilon;
  d.init_mode = p.init_mode;
  d.range = p.range;
  d.irls_tol = p.irls_tol;
  d.nlm_ratio = 0;
  return d;
}

int64_t mirror_host(int64_t i, int64_t n) {
  if (n == 1) return 0;
  const int64_t period = 2 * (n - 1);
  int64_t m = i % period;
  if (m < 0) m += period;
  return m < n ? m : period - m;
}

}  // namespace

extern "C" {

nlem_status nlem_frames_psnr(const float* frames, const float* clean, int64_t nframes,
                             int64_t count, double* psnr_out, nlem_failure* failure, void* stream) {
  clear(failure);
  if (nframes < 0 || count < 1) return invalid(failure, "psnr needs non-empty frames");
  if (nframes == 0) return NLEM_OK;
  if (!frames || !clean || !psnr_out) return invalid(failure, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* sse = nullptr;
  cudaError_t e = cudaMallocAsync(&sse, sizeof(double) * nframes, s);
  if (e == cudaSuccess) e = launch_frames_sse(frames, clean, nframes, count, sse, s);
  std::vector<double> h(static_cast<size_t>(nframes));
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), sse, sizeof(double) * nframes, cudaMemcpyDeviceToHost, s);
  if (sse) cudaFreeAsync(sse, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(failure, e);
  for (int64_t t = 0; t < nframes; ++t) {  // psnr.hpp:20-24
    const double mse = h[t] / static_cast<double>(count);
    psnr_out[t] = mse == 0.0 ? HUGE_VAL : 10.0 * std::log10(255.0 * 255.0 / mse);
  }
  return NLEM_OK;
}

nlem_status nlem_optimality_residual_batched(const float* points, const float* weights,
                                             int64_t batch, int64_t n, int64_t d, nlem_box box,
                                             const float* z, float* residual_out,
                                             nlem_failure* failure, void* stream) {
  clear(failure);
  if (batch < 0) return invalid(failure, "batch must be nonnegative");
  if (n < 1) return invalid(failure, "point set must contain at least one point");
  if (d < 1 || d > kMaxDim) return invalid(failure, "point dimension must be in [1, 1024]");
  if (nlem_status st = check_box(box, failure)) return st;
  if (batch == 0) return NLEM_OK;
  if (!points || !weights || !z || !residual_out) return invalid(failure, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (failure) {
    if (nlem_status st = validate_points_dev(points, weights, batch, static_cast<int>(n),
                                             static_cast<int>(d), failure, s))
      return st;
  }
  cudaError_t e = launch_optimality(points, weights, z, batch, static_cast<int>(n),
                                    static_cast<int>(d), box, residual_out, s);
  if (e == cudaSuccess && failure) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(failure, e);
  return NLEM_OK;
}

const char* nlem_version(void) { return "nlem_b200 0.1 (sm_100a)"; }

const char* nlem_status_string(nlem_status s) {
  switch (s) {
    case NLEM_OK: return "ok";
    case NLEM_INVALID_ARGUMENT: return "invalid argument";
    case NLEM_NUMERIC_FAILURE: return "numeric failure";
    case NLEM_CUDA_ERROR: return "CUDA error";
  }
  return "unknown";
}

nlem_status nlem_validate_params(const nlem_params* params, nlem_failure* failure) {
  clear(failure);
  return validate_params_impl(params, failure);
}

int32_t nlem_default_init_mode(float sigma) {  // proj/src/nlm.cpp:13-15
  return sigma <= 60.0f ? NLEM_INIT_NOISY_PATCH : NLEM_INIT_NLM_PATCH;
}

int64_t nlem_band_halo(const nlem_params* p) { return p->search / 2 + p->patch / 2; }

nlem_status nlem_admm_batched(const float* points, const float* weights, int64_t batch, int64_t n,
                              int64_t d, const float* z_init, nlem_box box, nlem_admm_config cfg,
                              float* z_out, float* objective_out, int32_t* iters_out,
                              float* trace_objective, float* trace_residual, nlem_failure* failure,
                              void* stream) {
  clear(failure);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (batch < 0) return invalid(failure, "batch must be nonnegative");
  if (n < 1) return invalid(failure, "point set must contain at least one point");
  if (d < 1 || d > kMaxDim) return invalid(failure, "point dimension must be in [1, 1024]");
  if (!(cfg.mu > 0.0f)) return invalid(failure, "penalty mu must be positive");  // admm.hpp:30-34
  if (cfg.max_iter < 1) return invalid(failure, "max_iter must be at least 1");
  if (nlem_status st = check_box(box, failure)) return st;
  if (batch == 0) return NLEM_OK;
  if (!points || !weights || !z_out) return invalid(failure, "null buffer");
  if (n * d > (int64_t(1) << 31)) return invalid(failure, "point set too large");
  AdmmLaunch L{points, weights, batch, static_cast<int>(n), static_cast<int>(d), z_init, box,
               cfg.mu, cfg.max_iter, cfg.tol_primal,
               res_mode_for(cfg.tol_primal, trace_residual != nullptr), z_out, objective_out,
               iters_out, trace_objective, trace_residual, nullptr};
  // NLEM_BATCHED_KERNEL=fast|generic forces a kernel family (A/B measurements, tests; read per
  // call); the default is the best specialised kernel for the shape
  const char* force = std::getenv("NLEM_BATCHED_KERNEL");
  const std::string fk = force ? force : "";
  const bool lr = fk.empty() && admm_lr_supported(L);
  // validation: fused into the low-rank kernel (no extra pass over the points), else separate
  DevSlot inval(s);
  if (failure && lr) {
    const cudaError_t ei = inval.init();
    if (ei != cudaSuccess) return cuda_fail(failure, ei);
    L.invalid = inval.ptr;
  } else if (failure) {
    if (nlem_status st = validate_points_dev(points, weights, batch, static_cast<int>(n),
                                             static_cast<int>(d), failure, s))
      return st;
  }
  DevSlot slot(s);
  cudaError_t e = slot.init();
  if (e != cudaSuccess) return cuda_fail(failure, e);
  L.fail = reinterpret_cast<FailureSlot*>(slot.ptr);
  if (lr) {
    // low-rank kernel, then the exact p-form kernel over the problems it handed off
    int* scratch = nullptr;  // [0] hand-off count, [1] small-mu probe, [2..] hand-off list
    e = cudaMallocAsync(&scratch, (2 + batch) * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(scratch, 0, 2 * sizeof(int), s);
    if (e == cudaSuccess) e = launch_admm_lr(L, scratch + 2, scratch, scratch + 1, s);
    if (e == cudaSuccess) e = launch_admm_fast_list(L, scratch + 2, scratch, s);
    const bool stats = std::getenv("NLEM_LR_STATS") != nullptr;  // read per call (tests)
    if (stats && e == cudaSuccess) {  // diagnostics only: synchronises the stream
      int handed = 0;
      e = cudaMemcpyAsync(&handed, scratch, sizeof(int), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      std::fprintf(stderr, "admm_lr: %lld problems, %d handed to the p-form kernel\n",
                   static_cast<long long>(batch), handed);
    }
    if (scratch) {
      const cudaError_t ef = cudaFreeAsync(scratch, s);
      if (e == cudaSuccess) e = ef;
    }
  } else {
    e = fk != "generic" && admm_fast_supported(L) ? launch_admm_fast(L, s) : launch_admm_generic(L, s);
  }
  // Collinear point sets (affine rank 1) are one-dimensional problems: with tol 0 their exact
  // residual stop is reachable (as for d <= 16) and only the reference-form sweep reproduces
  // the reference's iteration count.  The p-form kernels above cannot tell, so such problems
  // are re-solved in reference form.  Only the iteration count / trace length can differ (the
  // iterate is at a fixed point after an exact stop), so this runs when they are requested.
  if (e == cudaSuccess && L.res_mode == RES_EXACT0 && !use_ref_form(L.n, L.d) &&
      (iters_out != nullptr || trace_objective != nullptr)) {
    int* cl = nullptr;  // [0] count, [1..] problem list
    e = cudaMallocAsync(&cl, (1 + batch) * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cl, 0, sizeof(int), s);
    if (e == cudaSuccess) e = launch_collinear(points, batch, L.n, L.d, cl + 1, cl, s);
    if (e == cudaSuccess) e = launch_admm_generic(L, s, cl + 1, cl, true);
    if (cl) {
      const cudaError_t ef = cudaFreeAsync(cl, s);
      if (e == cudaSuccess) e = ef;
    }
  }
  if (e != cudaSuccess) return cuda_fail(failure, e);
  if (!failure) return NLEM_OK;
  if (L.invalid) {  // an invalid input outranks any numeric failure of the same call
    unsigned long long iv = ~0ull;
    if ((e = inval.read(&iv)) != cudaSuccess) return cuda_fail(failure, e);
    if (nlem_status st = report_invalid(iv, failure)) return st;
  }
  unsigned long long v = ~0ull;
  if ((e = slot.read(&v)) != cudaSuccess) return cuda_fail(failure, e);
  return decode_failure(v, failure, 0);
}

nlem_status nlem_irls_batched(const float* points, const float* weights, int64_t batch, int64_t n,
                              int64_t d, const float* x_init, nlem_irls_config cfg, float* x_out,
                              float* objective_out, int32_t* iters_out, float* trace_objective,
                              nlem_failure* failure, void* stream) {
  clear(failure);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (batch < 0) return invalid(failure, "batch must be nonnegative");
  if (n < 1) return invalid(failure, "point set must contain at least one point");
  if (d < 1 || d > kMaxDim) return invalid(failure, "point dimension must be in [1, 1024]");
  if (!(cfg.epsilon > 0.0f)) return invalid(failure, "epsilon must be positive");  // irls.hpp:24-28
  if (cfg.max_iter < 1) return invalid(failure, "max_iter must be at least 1");
  if (batch == 0) return NLEM_OK;
  if (!points || !weights || !x_out) return invalid(failure, "null buffer");
  IrlsLaunch L{points, weights, batch, static_cast<int>(n), static_cast<int>(d), x_init,
               cfg.epsilon, cfg.max_iter, cfg.tol, x_out, objective_out, iters_out,
               trace_objective, nullptr};
  const bool reg = irls_reg_supported(L);
  DevSlot inval(s);  // validation fused into the register kernel, else a separate pass
  if (failure && reg) {
    const cudaError_t ei = inval.init();
    if (ei != cudaSuccess) return cuda_fail(failure, ei);
    L.invalid = inval.ptr;
  } else if (failure) {
    if (nlem_status st = validate_points_dev(points, weights, batch, static_cast<int>(n),
                                             static_cast<int>(d), failure, s))
      return st;
  }
  DevSlot slot(s);
  cudaError_t e = slot.init();
  if (e != cudaSuccess) return cuda_fail(failure, e);
  L.fail = reinterpret_cast<FailureSlot*>(slot.ptr);
  e = reg ? launch_irls_reg(L, s) : launch_irls_generic(L, s);
  if (e != cudaSuccess) return cuda_fail(failure, e);
  if (!failure) return NLEM_OK;
  if (L.invalid) {  // an invalid input outranks any numeric failure of the same call
    unsigned long long iv = ~0ull;
    if ((e = inval.read(&iv)) != cudaSuccess) return cuda_fail(failure, e);
    if (nlem_status st = report_invalid(iv, failure)) return st;
  }
  unsigned long long v = ~0ull;
  if ((e = slot.read(&v)) != cudaSuccess) return cuda_fail(failure, e);
  return decode_failure(v, failure, 0);
}

}  // extern "C"

namespace {

nlem_status denoise_rows_impl(const float* noisy, int64_t in_row0, int64_t in_rows, int64_t rows,
                              int64_t cols, int64_t out_row0, int64_t out_rows,
                              const nlem_params* params, float* out, float* frames,
                              nlem_failure* failure, void* stream, int nlm_ratio) {
  clear(failure);
  (void)nlemk::device_caps();  // per-device setup (memory-pool policy) before the first allocation
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows < 1 || cols < 1) return invalid(failure, "image must be non-empty");  // image.hpp:15
  if (nlem_status st = validate_params_impl(params, failure)) return st;
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > rows)
    return invalid(failure, "output rows outside the image");
  if (in_row0 < 0 || in_rows < 1 || in_row0 + in_rows > rows)
    return invalid(failure, "input rows outside the image");
  if (out_rows == 0) return NLEM_OK;
  if (!noisy || !out) return invalid(failure, "null buffer");
  // The caller's band must cover the output rows and a halo of S/2 + k/2 rows (mirrored at the
  // image edges): every patch of the S x S window grid around each output pixel.
  const int hb = params->search / 2 + params->patch / 2;
  for (int64_t r = out_row0 - hb; r < out_row0 + out_rows + hb; ++r) {
    const int64_t g = mirror_host(r, rows);
    if (g < in_row0 || g >= in_row0 + in_rows)
      return invalid(failure, "input rows do not cover the band and its halo");
  }
  // Kernel choice: best specialised kernel for the shape; NLEM_KERNEL=lr|tile|fast|generic
  // forces one (A/B measurements, tests; falls back to generic when unsupported).
  enum class Kind { LR, TILE, FAST, GENERIC };
  Kind kind = Kind::GENERIC;
  {
    NlemLaunch probe{nullptr, 0, 0, cols + 26, rows, cols, out_row0, out_rows,
                     dev_params(*params), out, frames, nullptr};
    const char* force = std::getenv("NLEM_KERNEL");  // per call: tests switch it in-process
    const std::string k = force ? force : "";
    if ((k.empty() || k == "lr") && nlem_lr_supported(probe)) kind = Kind::LR;
    else if ((k.empty() || k == "tile") && nlem_tile_supported(probe)) kind = Kind::TILE;
    else if ((k.empty() || k == "fast") && nlem_fast_supported(probe)) kind = Kind::FAST;
  }
  // Mirror-padded band.  The low-rank / tile kernels address a fixed (S_grid + k - 1)^2 tile per
  // pixel and mask smaller windows inside their grid, so their border is the grid's; rows of
  // that border beyond the caller's halo are read by zero-weight points only (clamped copies).
  int border = hb;
  if (kind == Kind::LR || kind == Kind::TILE) {
    NlemLaunch probe{nullptr, 0, 0, cols + 26, rows, cols, out_row0, out_rows,
                     dev_params(*params), out, frames, nullptr};
    border = nlem_tile_grid(probe) / 2 + params->patch / 2;
  }
  const int64_t pad_row0 = out_row0 - border;
  const int64_t pad_rows = out_rows + 2 * border;
  const int64_t pad_cols = cols + 2 * border;
  if (failure) {  // image.hpp:16 over the rows this band reads
    DevSlot vs(s);
    cudaError_t e = vs.init();
    if (e == cudaSuccess) e = launch_validate_image(noisy, in_rows * cols, vs.ptr, s);
    unsigned long long v = ~0ull;
    if (e == cudaSuccess) e = vs.read(&v);
    if (e != cudaSuccess) return cuda_fail(failure, e);
    if (v != ~0ull) return invalid(failure, "image intensities must be finite");
  }
  float* pad = nullptr;
  cudaError_t e = cudaMallocAsync(&pad, pad_rows * pad_cols * sizeof(float), s);
  if (e != cudaSuccess) return cuda_fail(failure, e);
  DevSlot slot(s);
  e = slot.init();
  if (e == cudaSuccess)
    e = launch_pad_band(noisy, in_row0, in_rows, rows, cols, pad, pad_row0, pad_rows, pad_cols,
                        border, s);
  if (e == cudaSuccess) {
    NlemDevParams dp = dev_params(*params);
    dp.nlm_ratio = nlm_ratio;
    NlemLaunch L{pad, pad_row0, pad_rows, pad_cols, rows, cols, out_row0, out_rows,
                 dp, out, frames, reinterpret_cast<FailureSlot*>(slot.ptr)};
    if (kind == Kind::LR) {
      // low-rank kernel, then the exact tile kernel over the pixels it handed off
      // [0] work counter, [1] hand-off count (-1: all), [2, 3] small-mu probe, [4] work counter
      // of the ring-12 launch, [8..] hand-off list
      int* scratch = nullptr;
      const int64_t pixels = out_rows * cols;
      e = cudaMallocAsync(&scratch, (8 + pixels) * sizeof(int), s);
      if (e == cudaSuccess) e = cudaMemsetAsync(scratch, 0, 8 * sizeof(int), s);
      int* probe = nlem_lr_probe_wanted(L) ? scratch + 2 : nullptr;
      if (e == cudaSuccess) e = launch_nlem_lr(L, scratch + 8, scratch + 1, scratch, probe, s);
      // small-mu regime with up to kLrBigRing sweeps: the ring-12 build takes the band (it
      // returns at once when the probe did not find that regime)
      if (e == cudaSuccess && probe != nullptr && L.P.iters <= kLrBigRing)
        e = launch_nlem_lr_ring12(L, scratch + 8, scratch + 1, scratch + 4, probe, s);
      if (e == cudaSuccess) e = launch_nlem_tile_list(L, scratch + 8, scratch + 1, s);
      const bool stats = std::getenv("NLEM_LR_STATS") != nullptr;  // read per call (tests)
      if (stats && e == cudaSuccess) {  // diagnostics only: synchronises the stream
        int handed = 0;
        e = cudaMemcpyAsync(&handed, scratch + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        std::fprintf(stderr, "nlem_lr: %lld pixels, %lld handed to the tile kernel\n",
                     static_cast<long long>(pixels),
                     handed < 0 ? static_cast<long long>(pixels) : static_cast<long long>(handed));
      }
      if (scratch) {
        const cudaError_t ef = cudaFreeAsync(scratch, s);
        if (e == cudaSuccess) e = ef;
      }
    } else if (kind == Kind::TILE) e = launch_nlem_tile(L, s);
    else if (kind == Kind::FAST) e = launch_nlem_fast(L, s);
    else e = launch_nlem_generic(L, s);
  }
  cudaFreeAsync(pad, s);
  if (e != cudaSuccess) return cuda_fail(failure, e);
  if (!failure) return NLEM_OK;
  unsigned long long v = ~0ull;
  if ((e = slot.read(&v)) != cudaSuccess) return cuda_fail(failure, e);
  return decode_failure(v, failure, cols);
}

}  // namespace

extern "C" {

nlem_status nlem_denoise_rows(const float* noisy, int64_t in_row0, int64_t in_rows, int64_t rows,
                              int64_t cols, int64_t out_row0, int64_t out_rows,
                              const nlem_params* params, float* out, float* frames,
                              nlem_failure* failure, void* stream) {
  return denoise_rows_impl(noisy, in_row0, in_rows, rows, cols, out_row0, out_rows, params, out,
                           frames, failure, stream, 0);
}

nlem_status nlem_denoise(const float* noisy, int64_t rows, int64_t cols, const nlem_params* params,
                         float* out, float* frames, nlem_failure* failure, void* stream) {
  return nlem_denoise_rows(noisy, 0, rows, rows, cols, 0, rows, params, out, frames, failure,
                           stream);
}

nlem_status nlm_denoise(const float* noisy, int64_t rows, int64_t cols, const nlem_params* params,
                        float* out, nlem_failure* failure, void* stream) {
  if (params == nullptr) return invalid(failure, "params must not be null");
  nlem_params p = *params;
  p.solver = NLEM_SOLVER_NLM_ONLY;  // centre of the weighted-mean patch (test_denoise.cpp:228-240)
  return denoise_rows_impl(noisy, 0, rows, rows, cols, 0, rows, &p, out, nullptr, failure, stream,
                           1);
}

nlem_status nlem_admm_batched_host(const float* points, const float* weights, int64_t batch,
                                   int64_t n, int64_t d, const float* z_init, nlem_box box,
                                   nlem_admm_config cfg, float* z_out, float* objective_out,
                                   int32_t* iters_out, float* trace_objective,
                                   float* trace_residual, nlem_failure* failure, int32_t device) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  clear(f);
  if (batch <= 0 || n < 1 || d < 1)
    return nlem_admm_batched(nullptr, nullptr, batch, n, d, nullptr, box, cfg, nullptr, nullptr,
                             nullptr, nullptr, nullptr, f, nullptr);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(f, e);
  cudaStream_t s = cudaStreamPerThread;
  const size_t P = static_cast<size_t>(batch) * n * d, Wn = static_cast<size_t>(batch) * n,
               Z = static_cast<size_t>(batch) * d, Tn = static_cast<size_t>(batch) * cfg.max_iter;
  float *dp = nullptr, *dw = nullptr, *dzi = nullptr, *dz = nullptr, *dob = nullptr, *dto = nullptr,
        *dtr = nullptr;
  int32_t* dit = nullptr;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, bytes, s);
  };
  alloc(reinterpret_cast<void**>(&dp), P * 4);
  alloc(reinterpret_cast<void**>(&dw), Wn * 4);
  alloc(reinterpret_cast<void**>(&dz), Z * 4);
  if (z_init) alloc(reinterpret_cast<void**>(&dzi), Z * 4);
  if (objective_out) alloc(reinterpret_cast<void**>(&dob), batch * 4);
  if (iters_out) alloc(reinterpret_cast<void**>(&dit), batch * 4);
  if (trace_objective) alloc(reinterpret_cast<void**>(&dto), Tn * 4);
  if (trace_residual) alloc(reinterpret_cast<void**>(&dtr), Tn * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, points, P * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, weights, Wn * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && dzi) e = cudaMemcpyAsync(dzi, z_init, Z * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && dto) e = cudaMemcpyAsync(dto, trace_objective, Tn * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && dtr) e = cudaMemcpyAsync(dtr, trace_residual, Tn * 4, cudaMemcpyHostToDevice, s);
  nlem_status st = NLEM_OK;
  if (e == cudaSuccess)
    st = nlem_admm_batched(dp, dw, batch, n, d, dzi, box, cfg, dz, dob, dit, dto, dtr, f, s);
  if (e == cudaSuccess && st == NLEM_OK) {
    e = cudaMemcpyAsync(z_out, dz, Z * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dob) e = cudaMemcpyAsync(objective_out, dob, batch * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dit) e = cudaMemcpyAsync(iters_out, dit, batch * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dto) e = cudaMemcpyAsync(trace_objective, dto, Tn * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dtr) e = cudaMemcpyAsync(trace_residual, dtr, Tn * 4, cudaMemcpyDeviceToHost, s);
  }
  for (void* p : {static_cast<void*>(dp), static_cast<void*>(dw), static_cast<void*>(dzi),
                  static_cast<void*>(dz), static_cast<void*>(dob), static_cast<void*>(dit),
                  static_cast<void*>(dto), static_cast<void*>(dtr)})
    if (p) cudaFreeAsync(p, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(f, e);
  return st;
}

nlem_status nlem_irls_batched_host(const float* points, const float* weights, int64_t batch,
                                   int64_t n, int64_t d, const float* x_init, nlem_irls_config cfg,
                                   float* x_out, float* objective_out, int32_t* iters_out,
                                   float* trace_objective, nlem_failure* failure, int32_t device) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  clear(f);
  if (batch <= 0 || n < 1 || d < 1)
    return nlem_irls_batched(nullptr, nullptr, batch, n, d, nullptr, cfg, nullptr, nullptr, nullptr,
                             nullptr, f, nullptr);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(f, e);
  cudaStream_t s = cudaStreamPerThread;
  const size_t P = static_cast<size_t>(batch) * n * d, Wn = static_cast<size_t>(batch) * n,
               Z = static_cast<size_t>(batch) * d,
               Tn = static_cast<size_t>(batch) * std::max(cfg.max_iter, 1);
  float *dp = nullptr, *dw = nullptr, *dxi = nullptr, *dx = nullptr, *dob = nullptr, *dto = nullptr;
  int32_t* dit = nullptr;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, bytes, s);
  };
  alloc(reinterpret_cast<void**>(&dp), P * 4);
  alloc(reinterpret_cast<void**>(&dw), Wn * 4);
  alloc(reinterpret_cast<void**>(&dx), Z * 4);
  if (x_init) alloc(reinterpret_cast<void**>(&dxi), Z * 4);
  if (objective_out) alloc(reinterpret_cast<void**>(&dob), batch * 4);
  if (iters_out) alloc(reinterpret_cast<void**>(&dit), batch * 4);
  if (trace_objective) alloc(reinterpret_cast<void**>(&dto), Tn * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, points, P * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, weights, Wn * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && dxi) e = cudaMemcpyAsync(dxi, x_init, Z * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && dto) e = cudaMemcpyAsync(dto, trace_objective, Tn * 4, cudaMemcpyHostToDevice, s);
  nlem_status st = NLEM_OK;
  if (e == cudaSuccess) st = nlem_irls_batched(dp, dw, batch, n, d, dxi, cfg, dx, dob, dit, dto, f, s);
  if (e == cudaSuccess && st == NLEM_OK) {
    e = cudaMemcpyAsync(x_out, dx, Z * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dob) e = cudaMemcpyAsync(objective_out, dob, batch * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dit) e = cudaMemcpyAsync(iters_out, dit, batch * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && dto) e = cudaMemcpyAsync(trace_objective, dto, Tn * 4, cudaMemcpyDeviceToHost, s);
  }
  for (void* p : {static_cast<void*>(dp), static_cast<void*>(dw), static_cast<void*>(dxi),
                  static_cast<void*>(dx), static_cast<void*>(dob), static_cast<void*>(dit),
                  static_cast<void*>(dto)})
    if (p) cudaFreeAsync(p, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(f, e);
  return st;
}

nlem_status nlem_denoise_rows_host(const float* noisy, int64_t in_row0, int64_t in_rows,
                                   int64_t rows, int64_t cols, int64_t out_row0, int64_t out_rows,
                                   const nlem_params* params, float* out, float* frames,
                                   nlem_failure* failure, int32_t device) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  clear(f);
  if (rows < 1 || cols < 1) return invalid(f, "image must be non-empty");
  if (nlem_status st = validate_params_impl(params, f)) return st;
  if (in_rows < 1 || out_rows < 0) return invalid(f, "row range outside the image");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(f, e);
  cudaStream_t s = cudaStreamPerThread;
  const size_t in_px = static_cast<size_t>(in_rows) * cols;
  const size_t out_px = static_cast<size_t>(out_rows) * cols;
  const size_t fr = frames ? out_px * params->solver_iters : 0;
  float *din = nullptr, *dout = nullptr, *dfr = nullptr;
  e = cudaMallocAsync(&din, in_px * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dout, std::max<size_t>(out_px, 1) * 4, s);
  if (e == cudaSuccess && frames) e = cudaMallocAsync(&dfr, std::max<size_t>(fr, 1) * 4, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(din, noisy, in_px * 4, cudaMemcpyHostToDevice, s);
  nlem_status st = NLEM_OK;
  if (e == cudaSuccess)
    st = nlem_denoise_rows(din, in_row0, in_rows, rows, cols, out_row0, out_rows, params, dout, dfr,
                           f, s);
  if (e == cudaSuccess && st == NLEM_OK && out_px) {
    e = cudaMemcpyAsync(out, dout, out_px * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && frames) e = cudaMemcpyAsync(frames, dfr, fr * 4, cudaMemcpyDeviceToHost, s);
  }
  if (din) cudaFreeAsync(din, s);
  if (dout) cudaFreeAsync(dout, s);
  if (dfr) cudaFreeAsync(dfr, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(f, e);
  return st;
}

nlem_status nlem_denoise_host(const float* noisy, int64_t rows, int64_t cols,
                              const nlem_params* params, float* out, float* frames,
                              nlem_failure* failure, int32_t device) {
  return nlem_denoise_rows_host(noisy, 0, rows, rows, cols, 0, rows, params, out, frames, failure,
                                device);
}

nlem_status nlem_patch_stack_host(const float* image, int64_t rows, int64_t cols, int64_t row,
                                  int64_t col, int32_t search, int32_t patch, float h,
                                  float* patches_out, float* weights_out, int64_t* n_out,
                                  int64_t* self_column_out, nlem_failure* failure,
                                  int32_t device) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  clear(f);
  // patch.cpp:90-97 (validate_image, image.hpp:14-17, then the size and pixel checks)
  if (rows < 1 || cols < 1) return invalid(f, "image must be non-empty");
  if (!image || !patches_out || !weights_out || !n_out || !self_column_out)
    return invalid(f, "null buffer");
  for (int64_t i = 0; i < rows * cols; ++i)
    if (!std::isfinite(image[i])) return invalid(f, "image intensities must be finite");
  if (search < 1 || search % 2 == 0) return invalid(f, "search window must be odd and positive");
  if (patch < 1 || patch % 2 == 0) return invalid(f, "patch size must be odd and positive");
  if (row < 0 || row >= rows || col < 0 || col >= cols) return invalid(f, "pixel outside the image");
  if (!(h > 0.0f)) return invalid(f, "similarity bandwidth h must be positive");  // patch.cpp:54
  if (static_cast<int64_t>(patch) * patch > kMaxDim)
    return invalid(f, "patch dimension k*k above 1024 is not supported");
  const int64_t hs = search / 2;
  const int64_t r0 = std::max<int64_t>(0, row - hs), r1 = std::min<int64_t>(rows - 1, row + hs);
  const int64_t c0 = std::max<int64_t>(0, col - hs), c1 = std::min<int64_t>(cols - 1, col + hs);
  const int64_t n = (r1 - r0 + 1) * (c1 - c0 + 1), d = static_cast<int64_t>(patch) * patch;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(f, e);
  cudaStream_t s = cudaStreamPerThread;
  float *dimg = nullptr, *dp = nullptr, *dw = nullptr;
  e = cudaMallocAsync(&dimg, rows * cols * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dp, n * d * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dw, n * 4, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dimg, image, rows * cols * 4, cudaMemcpyHostToDevice, s);
  const double hh = static_cast<double>(h);
  if (e == cudaSuccess)
    e = launch_patch_stack(dimg, rows, cols, row, col, search, patch,
                           static_cast<float>(1.0 / (hh * hh)), dp, dw, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(patches_out, dp, n * d * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(weights_out, dw, n * 4, cudaMemcpyDeviceToHost, s);
  for (void* p : {static_cast<void*>(dimg), static_cast<void*>(dp), static_cast<void*>(dw)})
    if (p) cudaFreeAsync(p, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(f, e);
  *n_out = n;
  *self_column_out = (row - r0) * (c1 - c0 + 1) + (col - c0);
  return NLEM_OK;
}

nlem_status nlem_solve_patch_host(const float* patches, const float* weights, int64_t n, int64_t d,
                                  int64_t self_column, const nlem_params* params, float* init_out,
                                  float* patch_out, nlem_failure* failure, int32_t device) {
  nlem_failure local;
  nlem_failure* f = failure ? failure : &local;
  clear(f);
  if (nlem_status st = validate_params_impl(params, f)) return st;
  if (n < 1) return invalid(f, "point set must contain at least one point");
  if (d < 1 || d > kMaxDim) return invalid(f, "point dimension must be in [1, 1024]");
  if (self_column < 0 || self_column >= n)  // nlem.cpp:13-15
    return invalid(f, "patch stack has no valid self column");
  if (!patches || !weights || !init_out || !patch_out) return invalid(f, "null buffer");
  if (n * d > (int64_t(1) << 31)) return invalid(f, "point set too large");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(f, e);
  cudaStream_t s = cudaStreamPerThread;
  float *dp = nullptr, *dw = nullptr, *dinit = nullptr, *dout = nullptr;
  e = cudaMallocAsync(&dp, n * d * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dw, n * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dinit, d * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dout, d * 4, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, patches, n * d * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, weights, n * 4, cudaMemcpyHostToDevice, s);
  nlem_status st = NLEM_OK;
  const bool nlm_only = params->solver == NLEM_SOLVER_NLM_ONLY;
  // NlmOnly builds no PointSet in the reference (nlem.cpp:26-31), so its inputs are not
  // validated; the solvers validate theirs (types.hpp:58-68)
  if (e == cudaSuccess && st == NLEM_OK)
    e = launch_initial_patch(dp, dw, static_cast<int>(n), static_cast<int>(d),
                             static_cast<int>(self_column), params->init_mode, params->range,
                             dinit, nlm_only ? dout : nullptr, s);
  if (e == cudaSuccess && st == NLEM_OK && !nlm_only) {
    if (params->solver == NLEM_SOLVER_ADMM) {  // nlem.cpp:35-43
      const nlem_admm_config c{params->mu, params->solver_iters, 0.0f};
      st = nlem_admm_batched(dp, dw, 1, n, d, dinit, params->range, c, dout, nullptr, nullptr,
                             nullptr, nullptr, f, s);
    } else {  // nlem.cpp:45-55: IRLS from the init, then the box projection
      const nlem_irls_config c{params->epsilon, params->solver_iters, params->irls_tol};
      st = nlem_irls_batched(dp, dw, 1, n, d, dinit, c, dout, nullptr, nullptr, nullptr, f, s);
      if (st == NLEM_OK) e = launch_clip(dout, static_cast<int>(d), params->range, s);
    }
  }
  if (e == cudaSuccess && st == NLEM_OK) {
    e = cudaMemcpyAsync(init_out, dinit, d * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(patch_out, dout, d * 4, cudaMemcpyDeviceToHost, s);
  }
  for (void* p : {static_cast<void*>(dp), static_cast<void*>(dw), static_cast<void*>(dinit),
                  static_cast<void*>(dout)})
    if (p) cudaFreeAsync(p, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(f, e);
  return st;
}

}  // extern "C"
