// Low-rank (Gram-form) EM-ADMM for batched standalone solves, d = 49, 3 <= n <= 448
// (BASELINE config 1: 65,536 problems x n = 441 x d = 49).
//
// Algebra: the p-form of admm.hpp:49-78 unrolled as in kernels_nlem_lr.cu.  With everything
// centred on m = z_0 (the initial consensus: the weighted mean, admm.hpp:40, or z_init),
//     s_k p_k = sum_r al_r c~_{t-r} - ga a~_k,     a~ = a - m,  c~ = c - m,
// so a point carries 8 scalars (H = ||s p - a~||^2, K = <s p - a~, a~>, ga, ||a~||^2, al_0..3)
// and a sweep is one dot product D_k = <a~_k, c~_t> plus one weighted sum sum_k ga'_k a~_k:
//     N = H + 2 (sum_r al_r <c~_{t-1-r}, c~_t> - (ga + 1) D) + ||c~_t||^2        (= ||p_k||^2)
//     s = min(1, lambda rsqrt N), B = K + D, H' = s (s N - 2B) + ||a~||^2, K' = s B - ||a~||^2,
//     ga' = s (ga + 1), al' = (s, s al_0, s al_1, s al_2)
//     z_t = P_C(z_{t-1} - g/n),  g = sum_r (sum_k al'_r) c~_{t-r} - sum_k ga'_k a~_k,
//     c~_{t+1} = 2 z_t - z_{t-1} - m.
// A problem whose history ring would drop a term above FP32 rounding of p (2^-22 ||p||), whose
// ||p||^2 expansion cancels (N < 2^-8 (H + ||c~||^2)), whose points are all equal (the
// exact-stop case of admm.hpp:77, tested structurally by the p-form kernel), or that produces a
// non-finite value is handed, through a device-side list, to the exact p-form kernel
// (admm_batched_fast), which then owns its outputs and failure record.
//
// Mapping (B200): one problem per CTA of 14 point warps + 1 consensus warp, 1 CTA per SM.
//  * the centred points live in REGISTERS (the p-form kernel kept them in shared memory and
//    re-read them every sweep): groups of 8 lanes own 8 points, each lane 7 contiguous
//    coordinates (j = 7 g + i, d padded to 56) as float2 point pairs, so both passes are FFMA2;
//  * lane g of a group owns the scalar state of point slot g: reduce-scatter of the 8 dot
//    products in the group, scalar update, all-gather of ga';
//  * each point warp folds its 4 groups and writes one 64-column partial row (coordinates at
//    columns 8 g + i, history sums sum_k al'_r in columns 8 r + 7); after the CTA barrier the
//    consensus warp sums the 14 rows in a fixed tree, forms z_t and c~_{t+1}, publishes c~
//    (named barrier 1) and then the Gram row (named barrier 2), so the point warps' dot products
//    overlap the Gram reduction; ptxas moves arithmetic across bar.sync, so the order is pinned
//    with a shared-memory store before each wait and a reload after the arrive;
//  * the next problem's points and weights stream into a shared-memory staging buffer with
//    16-byte cp.async during the current problem's sweeps.
// The batched IRLS kernel (irls_batched_reg, below) reuses the layout and the consensus warp.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#ifdef NLEM_BLR_STAMPS
#include <cstdio>
#endif

#include "launch.h"

namespace nlemk {

namespace blr {

constexpr int D = 49, G = 8, J = 7, KP = G / 2;
constexpr int WARPS = 14;          // point warps
constexpr int CW = WARPS;          // the consensus warp (no points)
constexpr int NW = WARPS + 1, ALL = 32 * NW;
constexpr int GPW = 32 / G, NG = GPW * WARPS, NCAP = NG * G;  // 56 groups, 448 points
constexpr int R = 4;
// Column layout of every per-coordinate row (partials, c~, m): lane g of a group owns
// coordinates j = 7 g + i (i < 7) at columns 8 g + i; column 8 g + 7 carries the history sum
// sum_k al'_g for g < 4 (partial rows) and is 0 otherwise.
constexpr int RS = 64;
constexpr float kThr2 = 1.0f / 17592186044416.0f;  // (2^-22)^2: ring term below FP32 rounding
constexpr float kCancel = 1.0f / 256.0f;           // N below 2^-8 (H + ||c~||^2): cancellation
constexpr int kProbe = 64;                         // problems sampled by the small-mu probe
// shared memory (floats)
constexpr int SM_STAGE = 0;                      // raw points of the next problem (+4 shift)
constexpr int SM_WST = SM_STAGE + NCAP * D + 4;  // raw weights of the next problem (+4 shift)
constexpr int SM_RED = SM_WST + NCAP + 4;        // [WARPS][RS] per-warp partial rows
// Published rows (c~ / x, m) are read by every point lane as two 16-byte loads at column 8 g:
// columns 32..63 sit 4 floats further on (RSK = RS + 4), so lanes g and g + 4 hit distinct banks
// (one wavefront per load instead of two; these loads follow the row barrier on every warp).
constexpr int RSK = RS + 4;
constexpr int SM_CB = SM_RED + WARPS * RS;       // [RSK] c~ of the coming sweep (skewed)
constexpr int SM_MB = SM_CB + RSK;               // [RSK] m (centring), then z~ for the cost (skewed)
constexpr int SM_GR = SM_MB + RSK;               // [8] Gram row: G_0..G_3, ||c~||^2, ||c~_{t-4}||^2
constexpr int SM_SCAL = SM_GR + 8;               // [32] block-sum scratch
constexpr int SM_PIN = SM_SCAL + 32;             // [ALL] barrier-ordering scratch
constexpr int SM_TOTAL = SM_PIN + ALL;
constexpr size_t SMEM_BYTES = size_t(SM_TOTAL) * sizeof(float);
static_assert(NCAP >= 441, "config-1 capacity");
static_assert(SM_WST % 4 == 0 && SM_RED % 4 == 0 && SM_CB % 4 == 0 && SM_MB % 4 == 0 &&
              SM_GR % 4 == 0, "alignment");

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ float rsq(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
// named barriers: the consensus warp arrives, the other warps wait (count = all threads)
__device__ __forceinline__ void bar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(ALL) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(ALL) : "memory");
}
// Barriers only order memory operations: ptxas freely moves register arithmetic and shuffles
// across them.  To keep work on the intended side, a value is stored to / reloaded from shared
// memory at the barrier (a store cannot sink below it, a load cannot rise above it).
constexpr int BAR_C = 1, BAR_GRAM = 2;
#ifdef NLEM_BLR_STAMPS
#define BLR_STAMP(v) long long v = clock64()
#else
#define BLR_STAMP(v)
#endif

// element e of `src` lands at dst[shift(src) + e], shift = (src / 4) mod 4, so that global and
// shared addresses agree mod 16 and the interior moves as 16-byte cp.async
__device__ __forceinline__ int stage_shift(const float* src) {
  return static_cast<int>((reinterpret_cast<uintptr_t>(src) >> 2) & 3);
}
__device__ __forceinline__ void stage_copy(float* dst, const float* src, int total) {
  const int s0 = stage_shift(src);
  const int nch = (s0 + total + 3) >> 2;
  const float* base = src - s0;  // 16-byte aligned
  for (int c = threadIdx.x; c < nch; c += ALL) {
    const int e0 = 4 * c - s0;
    if (e0 >= 0 && e0 + 3 < total) {
      cp16(dst + 4 * c, base + 4 * c);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q;
        if (e >= 0 && e < total) cp4(dst + 4 * c + q, base + 4 * c + q);
      }
    }
  }
}

// Reduce-scatter of 8 per-point values (4 float2 slots) across the 8 lanes of a group: lane g
// returns the sum for point slot g.  Fixed tree (bitwise deterministic).
__device__ __forceinline__ float group_rs8(const float2 (&v)[KP], int g) {
  float x[G];
#pragma unroll
  for (int m = 0; m < KP; ++m) {
    x[2 * m] = v[m].x;
    x[2 * m + 1] = v[m].y;
  }
#pragma unroll
  for (int half = G / 2; half >= 1; half >>= 1) {
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
// All-gather of one value per lane of the group into 4 float2 slots (slot 2m, 2m+1).
__device__ __forceinline__ void group_ag8(float mine, float2 (&out)[KP], int lane) {
  const int base = lane & ~(G - 1);
#pragma unroll
  for (int m = 0; m < KP; ++m) {
    out[m].x = __shfl_sync(0xffffffffu, mine, base + 2 * m);
    out[m].y = __shfl_sync(0xffffffffu, mine, base + 2 * m + 1);
  }
}
// Sum the 7 per-lane column partials over the 4 groups of the warp (lanes of group 0 then
// hold the warp totals of their coordinates) and write them, with v7 in column 8 g + 7, as the
// warp's partial row (two 16-byte stores per lane of group 0).
__device__ __forceinline__ void fold_store(float (&v)[J], float v7, float* row, int lane) {
#pragma unroll
  for (int o = G; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < J; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane < G) {
    float4* d = reinterpret_cast<float4*>(row + 8 * lane);
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v7);
  }
}
// Column pair (2 lane, 2 lane + 1) summed over the WARPS partial rows in a fixed tree.
__device__ __forceinline__ float2 rows_sum(const float* red, int lane) {
  float2 r[WARPS];
#pragma unroll
  for (int w = 0; w < WARPS; ++w) r[w] = reinterpret_cast<const float2*>(red + w * RS)[lane];
#pragma unroll
  for (int span = 1; span < WARPS; span <<= 1)
#pragma unroll
    for (int w = 0; w + span < WARPS; w += 2 * span) r[w] = __fadd2_rn(r[w], r[w + span]);
  return r[0];
}
// columns 2 l, 2 l + 1 of a published row: the consensus lane l's pair.  SKEW (ADMM): columns
// 32..63 4 floats on; the IRLS kernel measured 1.5 % slower with the skew and keeps the plain row.
template <bool SKEW = true>
__device__ __forceinline__ float2* pub_pair(float* row, int lane) {
  return reinterpret_cast<float2*>(row + 2 * lane + (SKEW ? ((lane >> 4) << 2) : 0));
}
// the 7 coordinates (8 columns) of lane g of a group from a published row
template <bool SKEW = true>
__device__ __forceinline__ void load_coords(const float* row, int g, float (&c)[J]) {
  const float* const base = row + 8 * g + (SKEW ? ((g >> 2) << 2) : 0);
  const float4 a = reinterpret_cast<const float4*>(base)[0];
  const float4 b = reinterpret_cast<const float4*>(base)[1];
  c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
  c[4] = b.x; c[5] = b.y; c[6] = b.z;
}
// Block sum of one value per thread (fixed order), valid in thread 0 only.  One barrier: the
// next write of `scal` happens after the next problem's top-of-loop barrier.
__device__ __forceinline__ float block_sum0(float v, float* scal, int warp, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) scal[warp] = v;
  __syncthreads();
  float t = 0.0f;
  if (threadIdx.x == 0)
#pragma unroll
    for (int w = 0; w < NW; ++w) t += scal[w];
  return t;
}

// Fused input validation (types.hpp:58-68, the checks validate_points_dev runs as a separate
// pass): every thread checks the coordinates and weights it loaded (padding slots hold finite 0),
// the lowest failing (problem << 2 | code) wins; code 1 coordinates, 2 weights, 3 no positive
// weight - the reference's order within a problem.  One extra barrier per problem.
__device__ __forceinline__ void check_problem(const float2 (&A)[KP][J], const float2 (&wq)[KP],
                                              int64_t b, unsigned long long* invalid) {
  if (invalid == nullptr) return;  // uniform
  bool bad_pt = false, bad_w = false, pos = false;
#pragma unroll
  for (int m = 0; m < KP; ++m) {
#pragma unroll
    for (int i = 0; i < J; ++i) bad_pt |= !isfinite(A[m][i].x) || !isfinite(A[m][i].y);
    bad_w |= !(isfinite(wq[m].x) && wq[m].x >= 0.0f) || !(isfinite(wq[m].y) && wq[m].y >= 0.0f);
    pos |= wq[m].x > 0.0f || wq[m].y > 0.0f;
  }
  const unsigned long long key = static_cast<unsigned long long>(b) << 2;
  if (bad_pt) atomicMin(invalid, key | 1ull);
  if (bad_w) atomicMin(invalid, key | 2ull);
  if (!__syncthreads_or(pos) && threadIdx.x == 0) atomicMin(invalid, key | 3ull);
}

// Weighted-mean numerator and denominator in one row pass (admm.hpp:40 / irls.hpp:32 with
// types.hpp:71-74): the point warps write sum_k w_k a_k per coordinate and the weight sum (column
// 7) into their partial rows; one barrier; the consensus warp divides (sum w a) / (sum w).
__device__ __forceinline__ void weighted_sum_rows(const float2 (&A)[KP][J], const float2 (&wq)[KP],
                                                  float* myrow, bool is_pts, int lane) {
  float v[J];
#pragma unroll
  for (int i = 0; i < J; ++i) {
    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int m = 0; m < KP; ++m) acc = __ffma2_rn(wq[m], A[m][i], acc);
    v[i] = acc.x + acc.y;
  }
  float ws = 0.0f;  // weights of this lane's group (same in its 8 lanes), then of the warp
#pragma unroll
  for (int m = 0; m < KP; ++m) ws += wq[m].x + wq[m].y;
  ws += __shfl_xor_sync(0xffffffffu, ws, 8);
  ws += __shfl_xor_sync(0xffffffffu, ws, 16);
  if (is_pts) fold_store(v, lane == 0 ? ws : 0.0f, myrow, lane);
  __syncthreads();
}

}  // namespace blr

using namespace blr;

__global__ void __launch_bounds__(ALL, 1)
admm_batched_lr(const float* __restrict__ points, const float* __restrict__ weights,
                int64_t batch, int n, const float* __restrict__ z_init, nlem_box box, float mu,
                int T, float* z_out, float* obj_out, int* iters_out, int* ho_list,
                int* ho_count, unsigned long long* invalid, const int* probe_count) {
  // probe_count (optional): predicted small-mu hand-offs of kProbe sampled problems
  // (small_mu_probe_kernel).  Above 90 % the whole batch is in the small-mu regime (lambda =
  // w/mu >= ||p||: prox scales of 1, no decaying history, a ring overflow after R sweeps), and
  // every problem goes to the exact kernel right after its fused input validation.  The
  // decision depends on the input only (deterministic).
  const int64_t pt = batch < kProbe ? batch : kProbe;
  const bool all_mode =
      probe_count != nullptr && 10 * static_cast<int64_t>(*static_cast<const volatile int*>(probe_count)) > 9 * pt;
  extern __shared__ __align__(16) float smem[];
  float* const stage = smem + SM_STAGE;
  float* const wst = smem + SM_WST;
  float* const red = smem + SM_RED;
  float* const cb = smem + SM_CB;
  float* const mb = smem + SM_MB;
  float* const gr = smem + SM_GR;
  float* const scal = smem + SM_SCAL;
  float* const pin = smem + SM_PIN;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31;
  const int g = lane & (G - 1);
  const int gid = warp * GPW + (lane >> 3);
  const bool is_pts = warp < WARPS;
  float* const myrow = red + (is_pts ? warp : 0) * RS;
  // point of slot q of this lane's group: pair m = q / 2 is point pair m * NG + gid
  auto point_of = [&](int q) { return 2 * ((q >> 1) * NG + gid) + (q & 1); };
  const int k_me = point_of(g);
  const bool real_me = is_pts && k_me < n;
  // consensus (warp CW): lane l finishes columns 2l, 2l+1 = coordinates cj, cj + 1
  const int cgrp = lane >> 2, cidx = 2 * (lane & 3);
  const int cj = 7 * cgrp + cidx;
  const bool cv0 = cgrp < 7, cv1 = cgrp < 7 && (lane & 3) != 3;
  const float inv_mu = 1.0f / mu;
  const float inv_n = 1.0f / static_cast<float>(n);
  const int nd = n * D;

#ifdef NLEM_BLR_STAMPS
  long long su_wait = 0, su_load = 0, su_pref = 0, su_init = 0, su_sw = 0, su_epi = 0, su_n = 0;
#endif
  int64_t b = blockIdx.x;
  if (b < batch) {
    stage_copy(stage, points + b * nd, nd);
    stage_copy(wst, weights + b * n, n);
  }
  cp_commit();

  for (; b < batch; b += gridDim.x) {
#ifdef NLEM_BLR_STAMPS
    const long long su_t0 = clock64();
#endif
    cp_wait_all();
    __syncthreads();
#ifdef NLEM_BLR_STAMPS
    const long long su_t1 = clock64(); su_wait += su_t1 - su_t0;
#endif
    // ---- this problem's points (raw) into registers, weights, all-equal test
    const float* const src = points + b * nd;
    const float* const st = stage + stage_shift(src);
    const float* const wv = wst + stage_shift(weights + b * n);
    float2 A[KP][J];
    float2 wq[KP];
    int neq = 0;
    const bool greal = is_pts && g < 7;  // lane g = 7 of a group: padding coordinates 49..55
    float r0[J];
#pragma unroll
    for (int i = 0; i < J; ++i) r0[i] = greal ? st[7 * g + i] : 0.0f;
#pragma unroll
    for (int m = 0; m < KP; ++m) {
      const int k0 = 2 * (m * NG + gid), k1 = k0 + 1;
      const bool h0 = greal && k0 < n, h1 = greal && k1 < n;
      wq[m] = make_float2(is_pts && k0 < n ? wv[k0] : 0.0f, is_pts && k1 < n ? wv[k1] : 0.0f);
      const float* p0 = st + k0 * D + 7 * g;
      const float* p1 = st + k1 * D + 7 * g;
#pragma unroll
      for (int i = 0; i < J; ++i) {
        const float v0 = h0 ? p0[i] : r0[i], v1 = h1 ? p1[i] : r0[i];
        neq |= (v0 != r0[i]) | (v1 != r0[i]);
        A[m][i] = make_float2(h0 ? v0 : 0.0f, h1 ? v1 : 0.0f);
      }
    }
    const float w_me = real_me ? wv[k_me] : 0.0f;
    check_problem(A, wq, b, invalid);
    const bool static_eq = !__syncthreads_or(neq);  // every thread is done with the stage
#ifdef NLEM_BLR_STAMPS
    const long long su_t2 = clock64(); su_load += su_t2 - su_t1;
#endif
    const int64_t bn = b + gridDim.x;
    if (bn < batch) {
      stage_copy(stage, points + bn * nd, nd);
      stage_copy(wst, weights + bn * n, n);
    }
    cp_commit();
    // exact stop possible (the p-form kernel decides it structurally), or the small-mu regime
    if (static_eq || all_mode) {
      if (tid == 0) ho_list[atomicAdd(ho_count, 1)] = static_cast<int>(b);
      continue;
    }

#ifdef NLEM_BLR_STAMPS
    const long long su_t3 = clock64(); su_pref += su_t3 - su_t2;
#endif
    // ---- z_0 = m: z_init, or the weighted mean points * (w / sum w) (admm.hpp:40, types.hpp:73)
    float m0 = 0.0f, m1 = 0.0f;  // consensus warp: m at coordinates cj, cj + 1
    if (z_init == nullptr) weighted_sum_rows(A, wq, myrow, is_pts, lane);
    if (warp == CW) {
      if (z_init != nullptr) {
        m0 = cv0 ? z_init[b * D + cj] : 0.0f;
        m1 = cv1 ? z_init[b * D + cj + 1] : 0.0f;
      } else {
        const float2 s = rows_sum(red, lane);
        const float W = __shfl_sync(0xffffffffu, s.y, 3);  // sum of the weights (column 7)
        m0 = cv0 ? s.x / W : 0.0f;
        m1 = cv1 ? s.y / W : 0.0f;
      }
      *pub_pair(mb, lane) = make_float2(m0, m1);
      *pub_pair(cb, lane) = make_float2(0.0f, 0.0f);  // c~_1 = z_0 - m = 0
      if (lane < 8) gr[lane] = 0.0f;
    }
    __syncthreads();
    // centre the points on m
    float2 nq[KP];
    {
      float mc[J];
      load_coords(mb, g, mc);
#pragma unroll
      for (int m = 0; m < KP; ++m) nq[m] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < J; ++i) {
#pragma unroll
        for (int m = 0; m < KP; ++m) {
          const int k0 = 2 * (m * NG + gid);
          const float2 a = A[m][i];
          A[m][i] = make_float2(greal && k0 < n ? a.x - mc[i] : 0.0f,
                                greal && k0 + 1 < n ? a.y - mc[i] : 0.0f);
          nq[m] = __ffma2_rn(A[m][i], A[m][i], nq[m]);
        }
      }
    }
    const float a2 = group_rs8(nq, g);  // ||a~||^2 of this lane's point
    // per-point state (own slot): p_1 = z_0 - a = -a~ (u = 0, admm.hpp:41)
    float H = a2, K = -a2, ga = 0.0f, al0 = 0.0f, al1 = 0.0f, al2 = 0.0f, al3 = 0.0f;
    const float lam = inv_mu * w_me;
    // consensus state (warp CW): z, history ring c~_{t-r} (r = 0..3) and its norms
    float z0 = m0, z1 = m1;
    float h0[R], h1[R], nr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) h0[r] = h1[r] = nr[r] = 0.0f;
    bool bad = false, ovf = false;
#ifdef NLEM_BLR_STAMPS
    long long st_wc = 0, st_wg = 0, st_a = 0, st_b1 = 0, st_cons = 0, st_q[6] = {0, 0, 0, 0, 0, 0};
#endif

#ifdef NLEM_BLR_STAMPS
    const long long su_t4 = clock64(); su_init += su_t4 - su_t3;
#endif
    for (int t = 1; t <= T; ++t) {
     if (is_pts) {
      // (1) D_k = <a~_k, c~_t>
      // c~_t is published by the consensus warp before its Gram row (named barriers): the dot
      // products overlap the Gram reduction
      BLR_STAMP(s0);
      if (t > 1) bar_sync(BAR_C);
      BLR_STAMP(s1);
      float cv[J];
      load_coords(cb, g, cv);
      float2 dq[KP];
#pragma unroll
      for (int m = 0; m < KP; ++m) dq[m] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < J; ++i)
#pragma unroll
        for (int m = 0; m < KP; ++m) dq[m] = __ffma2_rn(A[m][i], f2(cv[i]), dq[m]);
      BLR_STAMP(q0);
      const float Dk = group_rs8(dq, g);
      BLR_STAMP(q1);
      // (2) scalar update of this lane's point
      BLR_STAMP(s2);
      if (t > 1) {
        pin[tid] = Dk;  // the dot products and their reduction run before the wait
        bar_sync(BAR_GRAM);
      }
      BLR_STAMP(s3);
      const float4 gq4 = reinterpret_cast<const float4*>(gr)[0];
      const float2 gq2 = reinterpret_cast<const float2*>(gr)[2];
      const float Gnn = gq2.x, nrR = gq2.y;
      const float X = fmaf(al0, gq4.x, fmaf(al1, gq4.y, fmaf(al2, gq4.z, al3 * gq4.w)));
      const float gp1 = ga + 1.0f;
      const float HG = H + Gnn;
      const float N = fmaf(2.0f, fmaf(-gp1, Dk, X), HG);
      bad |= lam != 0.0f && !isfinite(N);
      const float Nc = fmaxf(N, 0.0f);
      const float s = lam != 0.0f ? fminf(1.0f, lam * rsq(Nc)) : 0.0f;
      const float Bk = K + Dk;
      const float ev = s * al3;
      ovf |= ev * ev * nrR > kThr2 * Nc;
      ovf |= lam != 0.0f && N < kCancel * HG;
      H = fmaf(s, fmaf(s, Nc, -2.0f * Bk), a2);
      K = fmaf(s, Bk, -a2);
      ga = s * gp1;
      al3 = s * al2;
      al2 = s * al1;
      al1 = s * al0;
      al0 = s;
      // (3) sum_k ga'_k a~_k per coordinate; history sums sum_k al'_r (onto lanes r = 0..3)
      BLR_STAMP(q2);
      float2 gq[KP];
      group_ag8(ga, gq, lane);
      BLR_STAMP(q3);
      float v[J];
#pragma unroll
      for (int i = 0; i < J; ++i) {
        float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int m = 0; m < KP; ++m) acc = __ffma2_rn(gq[m], A[m][i], acc);
        v[i] = acc.x + acc.y;
      }
      BLR_STAMP(q4);
      float hs;
      {
        const bool u2 = (lane & 2) != 0, u1 = (lane & 1) != 0;
        const float x0 = (u2 ? al2 : al0) + __shfl_xor_sync(0xffffffffu, u2 ? al0 : al2, 2);
        const float x1 = (u2 ? al3 : al1) + __shfl_xor_sync(0xffffffffu, u2 ? al1 : al3, 2);
        hs = (u1 ? x1 : x0) + __shfl_xor_sync(0xffffffffu, u1 ? x0 : x1, 1);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
      }
      fold_store(v, lane < 4 ? hs : 0.0f, myrow, lane);
      BLR_STAMP(s4);
      __syncthreads();
      BLR_STAMP(s5);
#ifdef NLEM_BLR_STAMPS
      st_wc += s1 - s0; st_wg += s3 - s2; st_a += (s4 - s1) - (s3 - s2); st_b1 += s5 - s4;
      st_q[0] += q0 - s1; st_q[1] += q1 - q0; st_q[2] += q2 - s3; st_q[3] += q3 - q2; st_q[4] += q4 - q3; st_q[5] += s4 - q4;
#endif
     } else {
      BLR_STAMP(s4);
      __syncthreads();
      BLR_STAMP(s5);
#ifdef NLEM_BLR_STAMPS
      st_b1 += s5 - s4;
#endif
      // (4) consensus (warp CW): z_t = P_C(z_{t-1} - g/n), c~_{t+1} = 2 z_t - z_{t-1} - m, and
      // the Gram row of sweep t+1
        const float2 S = rows_sum(red, lane);
        float As[R];
#pragma unroll
        for (int r = 0; r < R; ++r) As[r] = __shfl_sync(0xffffffffu, S.y, 4 * r + 3);
        float g0 = -S.x, g1 = -S.y;
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
          g0 = fmaf(As[r], h0[r], g0);
          g1 = fmaf(As[r], h1[r], g1);
        }
        const float zn0 = cv0 ? clamp_box(fmaf(-g0, inv_n, z0), box) : 0.0f;
        const float zn1 = cv1 ? clamp_box(fmaf(-g1, inv_n, z1), box) : 0.0f;
        bad |= !isfinite(zn0) || !isfinite(zn1);
        const float c0 = cv0 ? (2.0f * zn0 - z0) - m0 : 0.0f;
        const float c1 = cv1 ? (2.0f * zn1 - z1) - m1 : 0.0f;
        z0 = zn0;
        z1 = zn1;
        *pub_pair(cb, lane) = make_float2(c0, c1);
        __syncwarp();
        if (t < T) bar_arrive(BAR_C);
        const float2 cg = *pub_pair(cb, lane);  // Gram after the arrive
        const float c0g = cg.x, c1g = cg.y;
        float part[R + 1];
#pragma unroll
        for (int r = 0; r < R; ++r) part[r] = fmaf(h0[r], c0g, h1[r] * c1g);
        part[R] = fmaf(c0g, c0g, c1g * c1g);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int q = 0; q <= R; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
        const float nr3 = nr[R - 1];
#pragma unroll
        for (int r = R - 1; r > 0; --r) {
          h0[r] = h0[r - 1];
          h1[r] = h1[r - 1];
          nr[r] = nr[r - 1];
        }
        h0[0] = c0;
        h1[0] = c1;
        nr[0] = part[R];
        if (lane == 0) {
          reinterpret_cast<float4*>(gr)[0] = make_float4(part[0], part[1], part[2], part[3]);
          reinterpret_cast<float2*>(gr)[2] = make_float2(part[R], nr3);
        }
        __syncwarp();
        if (t < T) bar_arrive(BAR_GRAM);
#ifdef NLEM_BLR_STAMPS
        BLR_STAMP(s6);
        st_cons += s6 - s5;
#endif
     }
    }

#ifdef NLEM_BLR_STAMPS
    if (blockIdx.x == 0 && b < 3 * gridDim.x && (tid == 0 || tid == 32 || tid == CW * 32))
      printf("blr stamps warp %d T %d: wait_c %lld wait_gram %lld phaseA %lld wait_b1 %lld cons %lld (per sweep)\n",
             warp, T, st_wc / T, st_wg / T, st_a / T, st_b1 / T, st_cons / T);
    if (blockIdx.x == 0 && b < 3 * gridDim.x && tid == 32)
      printf("blr phaseA: dot %lld rs8 %lld scalar %lld ag8 %lld wsum %lld fold+hs+sts %lld\n", st_q[0] / T,
             st_q[1] / T, st_q[2] / T, st_q[3] / T, st_q[4] / T, st_q[5] / T);
#endif
#ifdef NLEM_BLR_STAMPS
    const long long su_t5 = clock64(); su_sw += su_t5 - su_t4;
#endif
    // ---- hand-off or outputs
    if (__syncthreads_or(bad || ovf)) {
      if (tid == 0) ho_list[atomicAdd(ho_count, 1)] = static_cast<int>(b);
      continue;
    }
    if (warp == CW) {
      if (cv0) z_out[b * D + cj] = z0;
      if (cv1) z_out[b * D + cj + 1] = z1;
    }
    if (iters_out != nullptr && tid == 0) iters_out[b] = T;
    if (obj_out != nullptr) {
      // em_cost(z) = sum_k w_k ||z - a_k|| (costs.hpp:13-20), z - a = (z - m) - a~
      if (warp == CW) *pub_pair(mb, lane) = make_float2(z0 - m0, z1 - m1);
      __syncthreads();
      float zc[J];
      load_coords(mb, g, zc);
      float2 dq[KP];
#pragma unroll
      for (int m = 0; m < KP; ++m) dq[m] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < J; ++i) {
        const bool jr = 7 * g + i < D;
#pragma unroll
        for (int m = 0; m < KP; ++m) {
          const float2 e = __fadd2_rn(f2(zc[i]), make_float2(-A[m][i].x, -A[m][i].y));
          const float2 em = jr ? e : make_float2(0.0f, 0.0f);
          dq[m] = __ffma2_rn(em, em, dq[m]);
        }
      }
      const float dist2 = group_rs8(dq, g);
      const float obj = block_sum0(real_me ? w_me * sqrtf(dist2) : 0.0f, scal, warp, lane);
      if (tid == 0) {
        obj_out[b] = obj;
        if (!isfinite(obj)) ho_list[atomicAdd(ho_count, 1)] = static_cast<int>(b);
      }
    }
#ifdef NLEM_BLR_STAMPS
    { const long long e_ = clock64(); su_epi += e_ - su_t5; ++su_n; }
#endif
  }
#ifdef NLEM_BLR_STAMPS
  if (blockIdx.x < 2 && (tid == 0 || tid == CW * 32) && su_n)
    printf("blr setup blk %d warp %d: problems %lld wait %lld load %lld prefetch %lld init %lld sweeps %lld epilogue %lld\n",
           blockIdx.x, warp, su_n, su_wait / su_n, su_load / su_n, su_pref / su_n, su_init / su_n,
           su_sw / su_n, su_epi / su_n);
#endif
  cp_wait_all();
}

// ---------------------------------------------------------------------------------------
// Batched IRLS (proj/include/nlem/irls.hpp:21-68), d = 49, 1 <= n <= 448: the same register
// layout and consensus warp, direct differences (exact near coincident points, where epsilon
// matters).  Pass p evaluates at x_p: per point D = ||x_p - a_k||^2 (FADD2 + FFMA2), root =
// sqrt(D + eps), beta = w / root, the surrogate term w root (costs.hpp:24-33) and the cost term
// w sqrt(D) (costs.hpp:13-20, the objective output at the final x); the point warps reduce
// sum beta a, sum beta, the surrogate and the cost; the consensus warp applies the stop rule
// (irls.hpp:58) and forms x_{p+1} = sum beta a / sum beta.  Failures are recorded as the
// generic kernel does (iteration and kind of irls.hpp:39, :50, :52, :65-66).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(ALL, 1)
irls_batched_reg(const float* __restrict__ points, const float* __restrict__ weights,
                 int64_t batch, int n, const float* __restrict__ x_init, float eps, int T,
                 float tol, float* x_out, float* obj_out, int* iters_out, float* tr_obj,
                 FailureSlot* fail, unsigned long long* invalid) {
  extern __shared__ __align__(16) float smem[];
  float* const stage = smem + SM_STAGE;
  float* const wst = smem + SM_WST;
  float* const red = smem + SM_RED;
  float* const cb = smem + SM_CB;  // x of the coming pass
  int* const ctl = reinterpret_cast<int*>(smem + SM_GR);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31;
  const int g = lane & (G - 1);
  const int gid = warp * GPW + (lane >> 3);
  const bool is_pts = warp < WARPS;
  float* const myrow = red + (is_pts ? warp : 0) * RS;
  auto point_of = [&](int q) { return 2 * ((q >> 1) * NG + gid) + (q & 1); };
  const int k_me = point_of(g);
  const bool real_me = is_pts && k_me < n;
  const int cgrp = lane >> 2, cidx = 2 * (lane & 3);
  const int cj = 7 * cgrp + cidx;
  const bool cv0 = cgrp < 7, cv1 = cgrp < 7 && (lane & 3) != 3;
  const int nd = n * D;

  int64_t b = blockIdx.x;
  if (b < batch) {
    stage_copy(stage, points + b * nd, nd);
    stage_copy(wst, weights + b * n, n);
  }
  cp_commit();

  for (; b < batch; b += gridDim.x) {
    cp_wait_all();
    __syncthreads();
    const float* const st = stage + stage_shift(points + b * nd);
    const float* const wv = wst + stage_shift(weights + b * n);
    const bool greal = is_pts && g < 7;
    float2 A[KP][J];
    float2 wq[KP];
#pragma unroll
    for (int m = 0; m < KP; ++m) {
      const int k0 = 2 * (m * NG + gid), k1 = k0 + 1;
      const bool h0 = greal && k0 < n, h1 = greal && k1 < n;
      wq[m] = make_float2(is_pts && k0 < n ? wv[k0] : 0.0f, is_pts && k1 < n ? wv[k1] : 0.0f);
      const float* p0 = st + k0 * D + 7 * g;
      const float* p1 = st + k1 * D + 7 * g;
#pragma unroll
      for (int i = 0; i < J; ++i) A[m][i] = make_float2(h0 ? p0[i] : 0.0f, h1 ? p1[i] : 0.0f);
    }
    const float w_me = real_me ? wv[k_me] : 0.0f;
    check_problem(A, wq, b, invalid);
    __syncthreads();  // every thread is done with the stage
    const int64_t bn = b + gridDim.x;
    if (bn < batch) {
      stage_copy(stage, points + bn * nd, nd);
      stage_copy(wst, weights + bn * n, n);
    }
    cp_commit();

    // ---- x_0: x_init, or the weighted mean points * (w / sum w) (irls.hpp:32, types.hpp:73)
    if (x_init == nullptr) weighted_sum_rows(A, wq, myrow, is_pts, lane);
    float x0 = 0.0f, x1 = 0.0f;  // consensus warp: x of the current pass at cj, cj + 1
    if (warp == CW) {
      if (x_init != nullptr) {
        x0 = cv0 ? x_init[b * D + cj] : 0.0f;
        x1 = cv1 ? x_init[b * D + cj + 1] : 0.0f;
      } else {
        const float2 s = rows_sum(red, lane);
        const float W = __shfl_sync(0xffffffffu, s.y, 3);  // sum of the weights (column 7)
        x0 = cv0 ? s.x / W : 0.0f;
        x1 = cv1 ? s.y / W : 0.0f;
      }
      *pub_pair<false>(cb, lane) = make_float2(x0, x1);
    }
    __syncthreads();

    float previous = 0.0f, obj = 0.0f;
    int iters = T, fail_iter = -1, fail_kind = 0;
    for (int p = 0;; ++p) {
      if (is_pts) {
        float xc[J];
        load_coords<false>(cb, g, xc);
        float2 dq[KP];
#pragma unroll
        for (int m = 0; m < KP; ++m) dq[m] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int i = 0; i < J; ++i) {
#pragma unroll
          for (int m = 0; m < KP; ++m) {
            // no mask for the padding coordinates of lanes g = 7: their points are 0 and x's
            // padding columns are written as exact zeros (cv0 / cv1), so e = 0 there
            const float2 e = __fadd2_rn(f2(xc[i]), make_float2(-A[m][i].x, -A[m][i].y));
            dq[m] = __ffma2_rn(e, e, dq[m]);
          }
        }
        const float d2 = group_rs8(dq, g);
        // irls.hpp:45-46 and costs.hpp:24-33 / :13-20 with one hardware reciprocal square root
        // per point each (rsqrt.approx: ~2 ulp, against an FP64 reference)
        const float s2 = d2 + eps;
        const float ri = rsq(s2);
        const float beta = real_me ? w_me * ri : 0.0f;
        const float sur = real_me ? w_me * (s2 * ri) : 0.0f;
        const float cost = real_me && d2 > 0.0f ? w_me * (d2 * rsq(d2)) : 0.0f;
        float2 bq[KP];
        group_ag8(beta, bq, lane);
        float v[J];
#pragma unroll
        for (int i = 0; i < J; ++i) {
          float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int m = 0; m < KP; ++m) acc = __ffma2_rn(bq[m], A[m][i], acc);
          v[i] = acc.x + acc.y;
        }
        float hs;  // warp sums of (beta, surrogate, cost, 0) onto lanes r = lane & 3
        {
          const bool u2 = (lane & 2) != 0, u1 = (lane & 1) != 0;
          const float x0_ = (u2 ? cost : beta) + __shfl_xor_sync(0xffffffffu, u2 ? beta : cost, 2);
          const float x1_ = (u2 ? 0.0f : sur) + __shfl_xor_sync(0xffffffffu, u2 ? sur : 0.0f, 2);
          hs = (u1 ? x1_ : x0_) + __shfl_xor_sync(0xffffffffu, u1 ? x0_ : x1_, 1);
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
        }
        fold_store(v, lane < 4 ? hs : 0.0f, myrow, lane);
      }
      __syncthreads();
      if (warp == CW) {
        const float2 S = rows_sum(red, lane);
        const float den = __shfl_sync(0xffffffffu, S.y, 3);
        const float cur = __shfl_sync(0xffffffffu, S.y, 7);
        const float cst = __shfl_sync(0xffffffffu, S.y, 11);
        int c = 0;  // 0 continue, 1 done, 2 failed
        bool next = false;
        if (!isfinite(cur)) {  // irls.hpp:39 (x_0) / :52 (x_p)
          fail_iter = p;
          fail_kind = NLEM_FAIL_IRLS_OBJECTIVE;
          c = 2;
        } else if (p == 0) {
          previous = cur;
          next = true;
        } else {
          if (tr_obj != nullptr && lane == 0) tr_obj[b * T + p - 1] = cur;
          if (previous - cur <= tol * fabsf(previous)) {  // irls.hpp:58
            iters = p;
            obj = cst;
            c = 1;
          } else if (p == T) {
            obj = cst;
            c = 1;
          } else {
            previous = cur;
            next = true;
          }
        }
        if (next) {  // x_{p+1} = sum beta a / sum beta (irls.hpp:48)
          const float rden = 1.0f / den;
          const float n0 = cv0 ? S.x * rden : 0.0f, n1 = cv1 ? S.y * rden : 0.0f;
          if (__any_sync(0xffffffffu, !isfinite(n0) || !isfinite(n1))) {  // irls.hpp:50
            fail_iter = p + 1;
            fail_kind = NLEM_FAIL_IRLS_ITERATE;
            c = 2;
          } else {
            x0 = n0;
            x1 = n1;
            *pub_pair<false>(cb, lane) = make_float2(x0, x1);
          }
        }
        if (lane == 0) *ctl = c;
      }
      __syncthreads();
      if (*ctl != 0) break;
    }
    if (warp == CW) {
      if (fail_iter >= 0) {
        if (lane == 0) record_failure(fail, b, fail_iter, fail_kind);
      } else {
        if (cv0) x_out[b * D + cj] = x0;
        if (cv1) x_out[b * D + cj + 1] = x1;
        if (lane == 0) {
          if (iters_out != nullptr) iters_out[b] = iters;
          if (obj_out != nullptr) {
            obj_out[b] = obj;
            if (!isfinite(obj)) record_failure(fail, b, iters, NLEM_FAIL_IRLS_OBJECTIVE);
          }
        }
      }
    }
  }
  cp_wait_all();
}

bool irls_reg_supported(const IrlsLaunch& L) {
  const char* force = std::getenv("NLEM_BATCHED");  // =fast: the generic IRLS kernel (A/B, tests)
  if (force != nullptr && std::string(force) != "lr") return false;
  return L.d == D && L.n >= 1 && L.n <= NCAP && L.batch < (int64_t(1) << 31) &&
         static_cast<int64_t>(L.n) * D < (int64_t(1) << 31) / 4;
}

cudaError_t launch_irls_reg(const IrlsLaunch& L, cudaStream_t stream) {
  auto kfn = irls_batched_reg;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(L.batch, device_caps().sms));
  kfn<<<static_cast<unsigned>(grid), ALL, SMEM_BYTES, stream>>>(
      L.points, L.weights, L.batch, L.n, L.x_init, L.eps, L.max_iter, L.tol, L.x_out, L.obj_out,
      L.iters_out, L.tr_obj, L.fail, L.invalid);
  return cudaGetLastError();
}

bool admm_lr_supported(const AdmmLaunch& L) {
  const char* force = std::getenv("NLEM_BATCHED");  // =fast forces the p-form kernel (A/B, tests)
  if (force != nullptr && std::string(force) != "lr") return false;
  return L.d == D && L.n >= 3 && L.n <= NCAP && L.res_mode != RES_FULL && L.tr_obj == nullptr &&
         L.tr_res == nullptr && L.batch < (int64_t(1) << 31) &&
         static_cast<int64_t>(L.n) * D < (int64_t(1) << 31) / 4;
}

// Small-mu probe (one CTA per sampled problem, kProbe problems spread over the batch): at
// sweep 1 the ADMM local copies start from p_k = z_0 - a_k, so point k's prox scale saturates
// (s_k = 1) iff lambda_k = w_k / mu >= ||z_0 - a_k||.  A problem counts when more than half of
// its points saturate (the test admm_batched_lr applied at sweep 1 in round 1).
__global__ void __launch_bounds__(256)
small_mu_probe_kernel(const float* __restrict__ points, const float* __restrict__ weights,
                      int64_t batch, int n, const float* __restrict__ z_init, float mu, int pn,
                      int* probe_count) {
  __shared__ float z0[D];
  __shared__ float part[8];
  __shared__ int sat;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * batch / pn;
  const float* a = points + b * n * D;
  const float* w = weights + b * n;
  if (threadIdx.x == 0) sat = 0;
  // z_0: z_init, or the weighted mean points * (w / sum w) (admm.hpp:40, types.hpp:73)
  float ws = 0.0f;
  for (int k = threadIdx.x; k < n; k += blockDim.x) ws += w[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
  if (lane == 0) part[warp] = ws;
  __syncthreads();
  float W = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) W += part[i];
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    float m = 0.0f;
    if (z_init != nullptr) {
      m = z_init[b * D + j];
    } else {
      for (int k = 0; k < n; ++k) m = fmaf(a[static_cast<int64_t>(k) * D + j], w[k] / W, m);
    }
    z0[j] = m;
  }
  __syncthreads();
  int cnt = 0;
  for (int k = warp; k < n; k += 8) {
    float s2 = 0.0f;
    for (int j = lane; j < D; j += 32) {
      const float e = z0[j] - a[static_cast<int64_t>(k) * D + j];
      s2 = fmaf(e, e, s2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const float lam = w[k] / mu;
    cnt += lam * lam >= s2 && lam > 0.0f;
  }
  if (lane == 0) atomicAdd(&sat, cnt);
  __syncthreads();
  if (threadIdx.x == 0 && 2 * sat > n) atomicAdd(probe_count, 1);
}

cudaError_t launch_admm_lr(const AdmmLaunch& L, int* ho_list, int* ho_count, int* probe,
                           cudaStream_t stream) {
  auto kfn = admm_batched_lr;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  if (probe != nullptr && L.max_iter > R) {
    const int pn = static_cast<int>(std::min<int64_t>(L.batch, kProbe));
    small_mu_probe_kernel<<<pn, 256, 0, stream>>>(L.points, L.weights, L.batch, L.n, L.z_init,
                                                  L.mu, pn, probe);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else {
    probe = nullptr;
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(L.batch, device_caps().sms));
  kfn<<<static_cast<unsigned>(grid), ALL, SMEM_BYTES, stream>>>(
      L.points, L.weights, L.batch, L.n, L.z_init, L.box, L.mu, L.max_iter, L.z_out, L.obj_out,
      L.iters_out, ho_list, ho_count, L.invalid, probe);
  return cudaGetLastError();
}

}  // namespace nlemk
