// Register-tiled EM-ADMM for the benchmark shapes (d = 49, n <= 448 and d = 25, n <= 128):
// the batched standalone solve (BASELINE config 1) and the fused per-pixel NLEM kernel
// (configs 0, 2, 3).
//
// Layout (one CTA per problem/pixel, persistent grid):
//  * points are split into lane groups of G lanes; a group owns K = G points, each of
//    its lanes owns J coordinates (j = i*G + g), so d is padded to DP = G*J;
//  * the p-form state p_kj (solver_generic.cuh) lives in REGISTERS as float2 pairs of
//    two points (k, k+1) so every element op is one packed FFMA2/FADD2 (sm_100a);
//  * the points a_kj live in shared memory as float2 pairs [pair][DP] (row stride DP,
//    chosen so a warp's LDS.64 is bank-conflict free);
//  * per sweep: (U) p' = s p + (c - a) and ||p'||^2 partials, (R) reduce-scatter of the
//    norms inside the G-lane group -> each lane computes one prox scale s, all-gather,
//    (G) g = sum_k s_k p_k partials, warp butterfly over groups, one CTA barrier,
//    DP threads finish g over warps and form z' = P_C(z - g/n), c = 2z' - z.
// FP32 pipe work is 4 ops per element per sweep (the algorithmic count is 12 flops).
#include <algorithm>

#include "launch.h"
#include "solver_generic.cuh"

namespace nlemk {

template <int D_, int G_, int J_, int WARPS_>
struct FastCfg {
  static constexpr int D = D_;
  static constexpr int G = G_;          // lanes per group
  static constexpr int J = J_;          // coordinates per lane
  static constexpr int WARPS = WARPS_;
  static constexpr int K = G;           // points per group
  static constexpr int KP = K / 2;      // point pairs per lane
  static constexpr int GPW = 32 / G;    // groups per warp
  static constexpr int NG = GPW * WARPS;
  static constexpr int NCAP = NG * K;   // point capacity
  static constexpr int NPAIRS = NCAP / 2;
  static constexpr int DP = G * J;      // padded dimension
  static constexpr int THREADS = 32 * WARPS;
  static_assert(G * J >= D, "padding");
  static_assert(G % 2 == 0 && 32 % G == 0, "group size");
  static_assert(DP <= THREADS, "one thread per coordinate in the consensus step");
  // threads cooperating on one coordinate in the consensus step (power of two)
  static constexpr int CPT = THREADS >= 8 * DP ? 8 : THREADS >= 4 * DP ? 4 : THREADS >= 2 * DP ? 2 : 1;
};

using CfgD49 = FastCfg<49, 8, 7, 14>;  // 448 threads, n <= 448
using CfgD25 = FastCfg<25, 4, 7, 4>;   // 128 threads, n <= 128

// Shared-memory carve-up (float units).
template <class C>
struct FastSmem {
  static constexpr int A = C::NPAIRS * C::DP * 2;  // float2 a[NPAIRS][DP]
  static constexpr int RED = C::WARPS * C::DP;     // per-warp column partials
  static constexpr int TOTAL = A + RED + 2 * C::DP /*c2*/ + 3 * C::DP /*z,zprev,a0*/ +
                               C::NCAP /*lam/w*/ + 64 /*scalars, flags*/ +
                               C::NCAP /*koff*/ + C::DP /*joff*/;
};

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// prox scale s_k (see prox_scale) with the hardware reciprocal square root: lambda/||p||
// capped at 1 (||p|| <= lambda lands exactly on a_k: s == 1), 0 for lambda == 0.
__device__ __forceinline__ float prox_scale_fast(float lam, float nrm2) {
  if (lam == 0.0f) return 0.0f;
  return fminf(1.0f, lam * rsqrtf(nrm2));
}

// Reduce-scatter of K = G per-point partial values across the G lanes of a group:
// on return lane g holds the full sum for point slot g.  v[m] holds slots (2m, 2m+1).
template <class C>
__device__ __forceinline__ float group_reduce_scatter(float2 (&v)[C::KP], int g) {
  constexpr int K = C::K;
  float x[K];
#pragma unroll
  for (int m = 0; m < C::KP; ++m) {
    x[2 * m] = v[m].x;
    x[2 * m + 1] = v[m].y;
  }
#pragma unroll
  for (int half = K / 2; half >= 1; half >>= 1) {
    const bool up = (g & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = up ? x[i + half] : x[i];
      const float send = up ? x[i] : x[i + half];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return x[0];
}

// All-gather of one value per lane of the group into K/2 float2 slots.
template <class C>
__device__ __forceinline__ void group_all_gather(float mine, float2 (&out)[C::KP], int lane) {
  const int base = lane & ~(C::G - 1);
#pragma unroll
  for (int m = 0; m < C::KP; ++m) {
    out[m].x = __shfl_sync(0xffffffffu, mine, base + 2 * m);
    out[m].y = __shfl_sync(0xffffffffu, mine, base + 2 * m + 1);
  }
}

// Sum per-lane column partials (column j = i*G + g) over the groups of the warp; group 0
// writes the warp's partial to red[warp][j].
template <class C>
__device__ __forceinline__ void warp_columns_to_smem(float (&v)[C::J], float* red, int warp,
                                                     int lane) {
#pragma unroll
  for (int o = C::G; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < C::J; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane < C::G)
#pragma unroll
    for (int i = 0; i < C::J; ++i) red[warp * C::DP + i * C::G + lane] = v[i];
}

// Per-thread register state + smem pointers of one CTA.
template <class C>
struct FastCore {
  float2* a2;     // [NPAIRS][DP]
  float* red;     // [WARPS][DP]
  float2* c2;     // [DP]
  float* z;       // [DP]
  float* zprev;   // [DP]
  float* a0;      // [DP]  point 0 (exact-stop test)
  float* lam;     // [NCAP] w_k (batched: weights; NLEM: similarity weights)
  float* scal;    // scalars / flags
  int* koff;      // [NCAP] NLEM: tile offset of window-grid point k
  int* joff;      // [DP]   NLEM: tile offset of patch coordinate j (-1 = padding)
  int tid, warp, lane, g, gid;

  __device__ void carve(float* smem) {
    a2 = reinterpret_cast<float2*>(smem);
    red = smem + FastSmem<C>::A;
    c2 = reinterpret_cast<float2*>(red + FastSmem<C>::RED);
    z = reinterpret_cast<float*>(c2 + C::DP);
    zprev = z + C::DP;
    a0 = zprev + C::DP;
    lam = a0 + C::DP;
    scal = lam + C::NCAP;
    koff = reinterpret_cast<int*>(scal + 64);
    joff = koff + C::NCAP;
    tid = threadIdx.x;
    warp = tid >> 5;
    lane = tid & 31;
    g = lane & (C::G - 1);
    gid = warp * C::GPW + lane / C::G;
  }
  __device__ __forceinline__ int pair_of(int m) const { return m * C::NG + gid; }
  __device__ __forceinline__ int point_of_slot(int slot) const {
    return 2 * pair_of(slot >> 1) + (slot & 1);
  }
  __device__ __forceinline__ float2 a_at(int m, int i) const {
    return a2[pair_of(m) * C::DP + i * C::G + g];
  }
};

// Column sums over all points of  coef_k * a_kj  (coef per point slot from the group),
// finished over warps by threads j < DP into out[j].  One barrier inside, one at the end.
template <class C>
__device__ void colsum_weighted_points(FastCore<C>& S, const float2 (&coef)[C::KP], float* out,
                                       float post_scale, bool divide) {
  float v[C::J];
#pragma unroll
  for (int i = 0; i < C::J; ++i) {
    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int m = 0; m < C::KP; ++m) acc = fma2(coef[m], S.a_at(m, i), acc);
    v[i] = acc.x + acc.y;
  }
  warp_columns_to_smem<C>(v, S.red, S.warp, S.lane);
  __syncthreads();
  if (S.tid < C::DP) {
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < C::WARPS; ++w) t += S.red[w * C::DP + S.tid];
    out[S.tid] = (S.tid < C::D) ? (divide ? t / post_scale : t) : 0.0f;
  }
  __syncthreads();
}

// Block sum of one scalar per (point slot owner lane): lanes hold values for distinct
// points; fixed order (shuffle tree in warp, then warps in order).
template <class C>
__device__ float block_sum_scalar(FastCore<C>& S, float v) {
  v = warp_sum(v);
  if (S.lane == 0) S.scal[32 + S.warp] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int w = 0; w < C::WARPS; ++w) t += S.scal[32 + w];
  __syncthreads();
  return t;
}

struct FastResult {
  int iterations;
  int fail_iter;
  int fail_kind;
};

// The sweep loop.  Preconditions (all visible after a barrier): a2/lam/a0 filled (lam = 0
// for padding points), z holds z0 (padded coordinates 0), `static_eq` = every real point
// equals point a0.  my_real: the point of this lane's slot is a real point; nf = #real.
// on_iter(t) is called by thread 0 after sweep t with S.z holding z_t.
template <class C, class OnIter>
__device__ FastResult fast_admm_sweeps(FastCore<C>& S, bool my_real, float nf, nlem_box box,
                                       float mu, int T, int res_mode, bool static_eq,
                                       OnIter on_iter) {
  const float inv_mu = 1.0f / mu;
  const float inv_n = 1.0f / nf;
  const int my_point = S.point_of_slot(S.g);
  const float my_lam = my_real ? inv_mu * S.lam[my_point] : 0.0f;
  int* flags = reinterpret_cast<int*>(S.scal);  // [0..1] per-parity flag words
  FastResult res{T, -1, 0};
  // consensus role: column cj, part cpart of CPT cooperating threads
  const int cj = S.tid / C::CPT, cpart = S.tid % C::CPT;

  float2 p[C::KP][C::J];
  float2 s2[C::KP];
  // first sweep's state: p = z0 - a  (u = 0, admm.hpp:41)
#pragma unroll
  for (int m = 0; m < C::KP; ++m) s2[m] = make_float2(0.0f, 0.0f);
  if (S.tid < C::DP) S.c2[S.tid] = f2(S.z[S.tid]);
  if (S.tid == 0) {
    flags[0] = 0;
    flags[1] = 0;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < C::KP; ++m)
#pragma unroll
    for (int i = 0; i < C::J; ++i) p[m][i] = make_float2(0.0f, 0.0f);

  for (int t = 1; t <= T; ++t) {
    // (U) p' = s p + (c - a), norm partials
    float2 nr[C::KP];
#pragma unroll
    for (int m = 0; m < C::KP; ++m) nr[m] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < C::J; ++i) {
      const float2 cc = S.c2[i * C::G + S.g];
#pragma unroll
      for (int m = 0; m < C::KP; ++m) {
        const float2 ca = sub2(cc, S.a_at(m, i));
        p[m][i] = fma2(s2[m], p[m][i], ca);
        nr[m] = fma2(p[m][i], p[m][i], nr[m]);
      }
    }
    // (R) norms -> this lane's prox scale -> all lanes of the group
    const float nrm2 = group_reduce_scatter<C>(nr, S.g);
    const float s_mine = prox_scale_fast(my_lam, nrm2);
    const bool my_ok = isfinite(nrm2);
    const bool my_one = !my_real || s_mine == 1.0f;
    group_all_gather<C>(s_mine, s2, S.lane);
    // (G) g_j partials
    float v[C::J];
#pragma unroll
    for (int i = 0; i < C::J; ++i) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int m = 0; m < C::KP; ++m) acc = fma2(s2[m], p[m][i], acc);
      v[i] = acc.x + acc.y;
    }
    warp_columns_to_smem<C>(v, S.red, S.warp, S.lane);
    const int wbad = __any_sync(0xffffffffu, !my_ok);
    const int wnot1 = __any_sync(0xffffffffu, !my_one);
    if (S.lane == 0 && (wbad | wnot1)) atomicOr(&flags[t & 1], (wbad ? 1 : 0) | (wnot1 ? 2 : 0));
    __syncthreads();
    // consensus z_t = P_C(z_{t-1} - g/n), c = 2 z_t - z_{t-1}  (admm.hpp:59-65 in p-form);
    // CPT threads per coordinate: strided partial sums over warps, then a lane butterfly
    if (S.tid == 0) flags[(t + 1) & 1] = 0;
    {
      float gs = 0.0f;
      if (cj < C::DP)
#pragma unroll
        for (int w = cpart; w < C::WARPS; w += C::CPT) gs += S.red[w * C::DP + cj];
#pragma unroll
      for (int o = 1; o < C::CPT; o <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
      if (cj < C::DP && cpart == 0) {
        const float zo = S.z[cj];
        float zn = 0.0f;
        int f = 0;
        if (cj < C::D) {
          zn = clamp_box(fmaf(-gs, inv_n, zo), box);
          f |= isfinite(zn) ? 0 : 4;
          f |= (zn != S.a0[cj]) ? 8 : 0;
        }
        S.z[cj] = zn;
        S.c2[cj] = f2(2.0f * zn - zo);
        if (f) atomicOr(&flags[t & 1], f);
      }
    }
    __syncthreads();
    const int fl = flags[t & 1];
    if (fl & (4 | 1)) {  // non-finite z_t, or a multiplier blow-up in sweep t-1
      res.fail_iter = (fl & 4) || t == 1 ? t : t - 1;
      res.fail_kind = NLEM_FAIL_ADMM_ITERATE;
      return res;
    }
    if (S.tid == 0) on_iter(t);
    if (res_mode == RES_EXACT0 && static_eq && !(fl & 2) && !(fl & 8)) {
      res.iterations = t;  // every x_k == a_k == z_t: residual exactly 0 (admm.hpp:77)
      return res;
    }
  }
  return res;
}

// em_cost(z) = sum_k w_k ||z - a_k|| over real points (costs.hpp:13-20).
template <class C>
__device__ float fast_em_cost(FastCore<C>& S, int n) {
  float2 d2[C::KP];
#pragma unroll
  for (int m = 0; m < C::KP; ++m) d2[m] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int i = 0; i < C::J; ++i) {
    const float2 zz = f2(S.z[i * C::G + S.g]);
#pragma unroll
    for (int m = 0; m < C::KP; ++m) {
      const float2 e = sub2(zz, S.a_at(m, i));
      d2[m] = fma2(e, e, d2[m]);
    }
  }
  const float mine = group_reduce_scatter<C>(d2, S.g);
  const int k = S.point_of_slot(S.g);
  const float term = k < n ? S.lam[k] * sqrtf(mine) : 0.0f;
  return block_sum_scalar<C>(S, term);
}

// ---------------------------------------------------------------------------------------
// Batched standalone solves (config 1)
// ---------------------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
admm_batched_fast(const float* __restrict__ points, const float* __restrict__ weights,
                  int64_t batch, int n, const float* __restrict__ z_init, nlem_box box, float mu,
                  int T, int res_mode, float* z_out, float* obj_out, int* iters_out,
                  FailureSlot* fail, const int* list, const int* list_count) {
  extern __shared__ __align__(16) float smem[];
  FastCore<C> S;
  S.carve(smem);
  const size_t nd = static_cast<size_t>(n) * C::D;
  // list mode: the problems handed off by the low-rank kernel (kernels_batched_lr.cu)
  const int64_t count = list != nullptr ? *list_count : batch;
  for (int64_t ib = blockIdx.x; ib < count; ib += gridDim.x) {
    const int64_t b = list != nullptr ? list[ib] : ib;
    const float* pts = points + b * nd;
    // a -> smem pairs (coalesced global reads along j)
    int neq = 0;
    for (int e = S.tid; e < C::NPAIRS * C::DP; e += C::THREADS) {
      const int kp = e / C::DP, j = e - kp * C::DP;
      const int k0 = 2 * kp, k1 = k0 + 1;
      float v0 = 0.0f, v1 = 0.0f;
      if (j < C::D) {
        if (k0 < n) v0 = __ldg(pts + static_cast<size_t>(k0) * C::D + j);
        if (k1 < n) v1 = __ldg(pts + static_cast<size_t>(k1) * C::D + j);
        const float r0 = __ldg(pts + j);
        neq |= (k0 < n && v0 != r0) | (k1 < n && v1 != r0);
      }
      S.a2[e] = make_float2(v0, v1);
    }
    for (int k = S.tid; k < C::NCAP; k += C::THREADS) S.lam[k] = k < n ? weights[b * n + k] : 0.0f;
    if (S.tid < C::DP) S.a0[S.tid] = S.tid < C::D ? __ldg(pts + S.tid) : 0.0f;
    const bool static_eq = !__syncthreads_or(neq);
    // z0: z_init or the weighted mean points * (w / sum w)  (admm.hpp:40, types.hpp:71-74)
    if (z_init != nullptr) {
      if (S.tid < C::DP) S.z[S.tid] = S.tid < C::D ? z_init[b * C::D + S.tid] : 0.0f;
      __syncthreads();
    } else if (n == 1) {
      if (S.tid < C::DP) S.z[S.tid] = S.a0[S.tid];
      __syncthreads();
    } else {
      const int ks = S.point_of_slot(S.g);
      const float W = block_sum_scalar<C>(S, ks < n ? S.lam[ks] : 0.0f);
      float2 coef[C::KP];
#pragma unroll
      for (int m = 0; m < C::KP; ++m) {
        const int k0 = 2 * S.pair_of(m);
        coef[m] = make_float2(k0 < n ? S.lam[k0] / W : 0.0f, k0 + 1 < n ? S.lam[k0 + 1] / W : 0.0f);
      }
      colsum_weighted_points<C>(S, coef, S.z, 1.0f, false);
    }
    const FastResult r = fast_admm_sweeps<C>(S, S.point_of_slot(S.g) < n, static_cast<float>(n),
                                             box, mu, T, res_mode, static_eq, [](int) {});
    if (r.fail_iter >= 0) {
      if (S.tid == 0) record_failure(fail, b, r.fail_iter, r.fail_kind);
      __syncthreads();
      continue;
    }
    if (S.tid < C::D) z_out[b * C::D + S.tid] = S.z[S.tid];
    if (iters_out != nullptr && S.tid == 0) iters_out[b] = r.iterations;
    if (obj_out != nullptr) {
      const float obj = fast_em_cost<C>(S, n);
      if (S.tid == 0) {
        obj_out[b] = obj;
        if (!isfinite(obj)) record_failure(fail, b, r.iterations, NLEM_FAIL_ADMM_OBJECTIVE);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// Fused NLEM per pixel (configs 0, 2, 3): window tile -> patch stack in smem -> weights ->
// init -> ADMM sweeps -> centre coordinate (+ frames).
// ---------------------------------------------------------------------------------------
constexpr int kTileMax = 32 * 32;  // (S + k - 1)^2 <= 27^2 for S=21, k=7

// The stack of every pixel is laid out on the FULL S x S window grid centred on the pixel
// (point k = gr*S + gc); grid points outside the image are padding (weight 0, not counted
// in n).  That keeps every per-pixel index a table lookup (koff/joff) and the self point
// fixed at the grid centre.  The reference enumerates the clipped window row-major
// (patch.cpp:72-85); only the summation order differs.
template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
nlem_pixels_fast(const float* __restrict__ pad, int64_t pad_row0, int64_t pad_cols, int64_t rows,
                 int64_t cols, int64_t out_row0, int64_t out_rows, NlemDevParams P, float* out,
                 float* frames, int* work_counter, int chunk, FailureSlot* fail) {
  extern __shared__ __align__(16) float smem[];
  FastCore<C> S;
  S.carve(smem);
  float* tile = smem + FastSmem<C>::TOTAL;
  __shared__ int next_chunk;
  const int k = P.patch, SW = P.search, hs = SW / 2;
  const int TW = SW + k - 1;  // tile side
  const int center = C::D / 2;
  const int self = hs * SW + hs;
  const int64_t plane = out_rows * cols;
  const int64_t nchunks = (plane + chunk - 1) / chunk;
  (void)pad_row0;
  // per-launch tables
  for (int kk = S.tid; kk < C::NCAP; kk += C::THREADS)
    S.koff[kk] = kk < SW * SW ? (kk / SW) * TW + (kk % SW) : 0;
  for (int j = S.tid; j < C::DP; j += C::THREADS) S.joff[j] = j < C::D ? (j / k) * TW + (j % k) : -1;
  const int my_k = S.point_of_slot(S.g);
  const int my_gr = my_k < SW * SW ? my_k / SW : -1, my_gc = my_k < SW * SW ? my_k % SW : -1;
  __syncthreads();
  for (;;) {
    if (S.tid == 0) next_chunk = atomicAdd(work_counter, 1);
    __syncthreads();
    const int64_t ch = next_chunk;
    __syncthreads();
    if (ch >= nchunks) break;
    const int64_t pix_end = (ch + 1) * chunk < plane ? (ch + 1) * chunk : plane;
    for (int64_t pix = ch * chunk; pix < pix_end; ++pix) {
      const int64_t r = out_row0 + pix / cols, c = pix % cols;
      // real part of the grid (clipped window, patch.cpp:72-76)
      const int gr0 = r < hs ? static_cast<int>(hs - r) : 0;
      const int gr1 = rows - 1 - r < hs ? static_cast<int>(hs + (rows - 1 - r)) : SW - 1;
      const int gc0 = c < hs ? static_cast<int>(hs - c) : 0;
      const int gc1 = cols - 1 - c < hs ? static_cast<int>(hs + (cols - 1 - c)) : SW - 1;
      const int n = (gr1 - gr0 + 1) * (gc1 - gc0 + 1);
      const bool my_real = my_gr >= gr0 && my_gr <= gr1 && my_gc >= gc0 && my_gc <= gc1;
      // tile = padded image rows r-hs-hk.., cols c-hs-hk.. (pad row 0 = out_row0-hs-hk)
      const float* src = pad + (r - out_row0) * pad_cols + c;
      for (int e = S.tid; e < TW * TW; e += C::THREADS) {
        const int tr = e / TW, tc = e - tr * TW;
        tile[e] = __ldg(src + tr * pad_cols + tc);
      }
      __syncthreads();
      // patch stack as point pairs; footprint-constancy test for the exact stop
      const float ref = tile[gr0 * TW + gc0];
      int neq = 0;
      for (int e = S.tid; e < TW * TW; e += C::THREADS) {
        const int tr = e / TW, tc = e - tr * TW;
        if (tr >= gr0 && tr <= gr1 + k - 1 && tc >= gc0 && tc <= gc1 + k - 1) neq |= tile[e] != ref;
      }
      for (int e = S.tid; e < C::NPAIRS * C::DP; e += C::THREADS) {
        const int kp = e / C::DP, j = e - kp * C::DP;
        const int jo = S.joff[j];
        const int2 ko = reinterpret_cast<const int2*>(S.koff)[kp];
        S.a2[e] = jo >= 0 ? make_float2(tile[ko.x + jo], tile[ko.y + jo]) : make_float2(0.0f, 0.0f);
      }
      if (S.tid < C::DP) S.a0[S.tid] = S.tid < C::D ? ref : 0.0f;
      const bool static_eq = !__syncthreads_or(neq);
      // similarity weights w_k = exp(-||P_k - P_self||^2 / h^2) (patch.cpp:52-61)
      {
        float2 d2[C::KP];
#pragma unroll
        for (int m = 0; m < C::KP; ++m) d2[m] = make_float2(0.0f, 0.0f);
        const int sp = self >> 1, sq = self & 1;
#pragma unroll
        for (int i = 0; i < C::J; ++i) {
          const float2 sv = S.a2[sp * C::DP + i * C::G + S.g];
          const float2 ss = f2(sq ? sv.y : sv.x);
#pragma unroll
          for (int m = 0; m < C::KP; ++m) {
            const float2 e = sub2(S.a_at(m, i), ss);
            d2[m] = fma2(e, e, d2[m]);
          }
        }
        const float dsum = group_reduce_scatter<C>(d2, S.g);
        S.lam[my_k] = my_real ? expf(-dsum * P.inv_h2) : 0.0f;
      }
      __syncthreads();
      // initial patch (nlem.cpp:13-18)
      const bool nlm_init = P.solver == NLEM_SOLVER_NLM_ONLY || P.init_mode == NLEM_INIT_NLM_PATCH;
      if (nlm_init) {
        const float W = block_sum_scalar<C>(S, S.lam[my_k]);
        float2 coef[C::KP];
        const bool ratio = P.nlm_ratio != 0;
#pragma unroll
        for (int m = 0; m < C::KP; ++m) {
          const float2 w = reinterpret_cast<const float2*>(S.lam)[S.pair_of(m)];
          coef[m] = ratio ? w : make_float2(w.x / W, w.y / W);
        }
        colsum_weighted_points<C>(S, coef, S.z, W, ratio);
      } else {
        if (S.tid < C::DP) {
          const int sp = self >> 1, sq = self & 1;
          const float2 sv = S.a2[sp * C::DP + S.tid];
          S.z[S.tid] = S.tid < C::D ? (sq ? sv.y : sv.x) : 0.0f;
        }
        __syncthreads();
      }
      int iters = P.iters;
      int fail_iter = -1, fail_kind = 0;
      const int64_t opix = pix;
      if (P.solver == NLEM_SOLVER_ADMM) {
        const FastResult fr = fast_admm_sweeps<C>(
            S, my_real, static_cast<float>(n), P.range, P.mu, P.iters, RES_EXACT0, static_eq,
            [&](int t) {
              if (frames) frames[static_cast<int64_t>(t - 1) * plane + opix] = S.z[center];
            });
        iters = fr.iterations;
        fail_iter = fr.fail_iter;
        fail_kind = fr.fail_kind;
      }
      if (S.tid == 0) {
        if (fail_iter >= 0) {
          record_failure(fail, r * cols + c, fail_iter, fail_kind);
        } else {
          float v = S.z[center];
          if (P.solver != NLEM_SOLVER_ADMM) v = clamp_box(v, P.range);  // NlmOnly (nlem.cpp:26-31)
          out[pix] = v;
          if (frames) {
            const int from = P.solver == NLEM_SOLVER_ADMM ? iters : 0;
            for (int t = from; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pix] = v;
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
namespace {

template <class C>
size_t fast_smem_bytes(bool tile) {
  return (FastSmem<C>::TOTAL + (tile ? kTileMax : 0)) * sizeof(float);
}

template <class C>
cudaError_t launch_batched(const AdmmLaunch& L, cudaStream_t stream, const int* list = nullptr,
                           const int* list_count = nullptr) {
  const size_t smem = fast_smem_bytes<C>(false);
  auto kfn = admm_batched_fast<C>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, C::THREADS, smem);
  const int64_t grid =
      std::max<int64_t>(1, std::min<int64_t>(L.batch, int64_t(device_caps().sms) * std::max(per_sm, 1)));
  kfn<<<static_cast<unsigned>(grid), C::THREADS, smem, stream>>>(
      L.points, L.weights, L.batch, L.n, L.z_init, L.box, L.mu, L.max_iter, L.res_mode, L.z_out,
      L.obj_out, L.iters_out, L.fail, list, list_count);
  return cudaGetLastError();
}

template <class C>
cudaError_t launch_pixels(const NlemLaunch& L, cudaStream_t stream) {
  const size_t smem = fast_smem_bytes<C>(true);
  auto kfn = nlem_pixels_fast<C>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, C::THREADS, smem);
  const int64_t pixels = L.out_rows * L.cols;
  const int64_t ctas = int64_t(device_caps().sms) * std::max(per_sm, 1);
  const int chunk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, pixels / (ctas * 4))));
  int* counter = nullptr;
  e = cudaMallocAsync(&counter, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(counter, 0, sizeof(int), stream);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctas, (pixels + chunk - 1) / chunk));
  kfn<<<static_cast<unsigned>(grid), C::THREADS, smem, stream>>>(
      L.pad, L.pad_row0, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out, L.frames,
      counter, chunk, L.fail);
  e = cudaGetLastError();
  cudaFreeAsync(counter, stream);
  return e;
}

}  // namespace

bool admm_fast_supported(const AdmmLaunch& L) {
  if (L.res_mode == RES_FULL || L.tr_obj != nullptr || L.tr_res != nullptr) return false;
  if (L.n < 3) return false;  // n <= 2: reference-form sweep (exact stops, use_ref_form)
  if (L.d == CfgD49::D && L.n <= CfgD49::NCAP) return true;
  if (L.d == CfgD25::D && L.n <= CfgD25::NCAP) return true;
  return false;
}

cudaError_t launch_admm_fast(const AdmmLaunch& L, cudaStream_t stream) {
  if (L.d == CfgD49::D) return launch_batched<CfgD49>(L, stream);
  return launch_batched<CfgD25>(L, stream);
}

cudaError_t launch_admm_fast_list(const AdmmLaunch& L, const int* list, const int* list_count,
                                  cudaStream_t stream) {
  if (L.d == CfgD49::D) return launch_batched<CfgD49>(L, stream, list, list_count);
  return launch_batched<CfgD25>(L, stream, list, list_count);
}

bool nlem_fast_supported(const NlemLaunch& L) {
  if (L.P.solver == NLEM_SOLVER_IRLS) return false;
  const int d = L.P.patch * L.P.patch, n = L.P.search * L.P.search;
  const int tile = (L.P.search + L.P.patch - 1) * (L.P.search + L.P.patch - 1);
  if (tile > kTileMax) return false;
  if (d == CfgD49::D && n <= CfgD49::NCAP) return true;
  if (d == CfgD25::D && n <= CfgD25::NCAP) return true;
  return false;
}

cudaError_t launch_nlem_fast(const NlemLaunch& L, cudaStream_t stream) {
  const int d = L.P.patch * L.P.patch;
  if (d == CfgD49::D) return launch_pixels<CfgD49>(L, stream);
  return launch_pixels<CfgD25>(L, stream);
}

}  // namespace nlemk
