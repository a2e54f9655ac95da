// Low-rank (Gram-form) EM-ADMM for batched standalone solves, d = 49, 3 <= n <= 448
// (BASELINE config 1: 65,536 problems x n = 441 x d = 49), and the batched IRLS comparator.
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
// Mapping (B200), round 2: TWO problems in flight per SM.  A sweep is a serial chain (dot
// products -> group reduction -> per-point scalar update -> weighted sum -> CTA reduction ->
// consensus -> next dot products); with one problem per SM (round 1: 14 point warps at 128
// registers, every warp in the same phase) the FMA pipe sat idle for most of the chain.  Now one
// problem is a CTA of 7 point warps + 1 consensus warp at 128 registers and two CTAs share an
// SM, so one problem's reductions and barriers overlap the other's FFMA2s, and one problem's
// setup (load, validation, weighted mean, centring) overlaps the other's sweeps.
//  * groups of 8 lanes own 16 points as 8 float2 point pairs, each lane 7 contiguous
//    coordinates (j = 7 g + i, d padded to 56), so both passes are FFMA2 on a point pair;
//    pairs 0..3 of a group live in REGISTERS (56 per lane), pairs 4..7 in TENSOR MEMORY (56
//    columns of the lane, one tcgen05.ld pass of 16 + 16 + 16 + 8 columns per MAC pass) - the
//    register file holds one problem per SM, so the second problem's worth of points sits in
//    TMEM, whose read path (~176 B/clk/SM measured, tools/tmem_bw.cu) is separate from the
//    shared-memory / shuffle data pipe that the reductions already load (a shared-memory
//    resident half measured that pipe at 68 % with no gain over one problem per SM);
//  * lane g of a group owns the scalar state of point slots g and 8 + g: reduce-scatter of the
//    dot products in the group, scalar updates, all-gather of ga';
//  * each point warp folds its 4 groups and writes one 64-column partial row (coordinates at
//    columns 8 g + i, history sums sum_k al'_r in columns 8 r + 7); after the CTA barrier the
//    consensus warp sums the 7 rows in a fixed tree, forms z_t and c~_{t+1}, publishes c~
//    (named barrier 1) and then the Gram row (named barrier 2), so the point warps' dot products
//    overlap the Gram reduction; ptxas moves arithmetic across bar.sync, so the order is pinned
//    with a shared-memory store before each wait and a reload after the arrive;
//  * the next problem's points and weights stream into a shared-memory staging buffer with
//    16-byte cp.async during the current problem's sweeps (88 KB per CTA).
// The batched IRLS kernel (irls_batched_reg, below) reuses the layout and the consensus warp.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "launch.h"
#include "tmem.cuh"

namespace nlemk {

namespace blr {

constexpr int D = 49, G = 8, J = 7;
constexpr int KR = 4, KS = 4, KP = KR + KS;  // float2 point pairs per group: registers, smem
constexpr int WARPS = 7;                     // point warps
constexpr int CW = WARPS;                    // the consensus warp (no points)
constexpr int NW = WARPS + 1, ALL = 32 * NW;
constexpr int GPW = 32 / G, NG = GPW * WARPS, NCAP = NG * 2 * KP;  // 28 groups, 448 points
constexpr int R = 4;
constexpr int TM_HALF = KS * J * 2;          // TMEM columns per lane: the second half of its points
constexpr int TM_WCOLS = 64;                 // column slice of one warp (warps w and w + 4 share lanes)
constexpr int TM_COLS = 128;                 // TMEM columns allocated per CTA
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
constexpr int SM_TB = SM_PIN + ALL;               // [4] TMEM base address of the CTA
constexpr int SM_TOTAL = SM_TB + 4;
constexpr size_t SMEM_BYTES = size_t(SM_TOTAL) * sizeof(float);
static_assert(NCAP >= 441, "config-1 capacity");
static_assert(TM_HALF == 56 && TM_HALF <= TM_WCOLS && 2 * TM_WCOLS <= TM_COLS, "TMEM layout");
static_assert(SM_WST % 4 == 0 && SM_RED % 4 == 0 && SM_CB % 4 == 0 && SM_MB % 4 == 0 && SM_GR % 4 == 0, "alignment");
static_assert(2 * (SMEM_BYTES + 1024) <= 233472, "two CTAs per SM");

__device__ __forceinline__ float rsq(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ void cp16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tm::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tm::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
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

// The TMEM-resident half of a lane's points: 56 columns holding the float2 point pairs of the
// sequence e = 0..27 (pair m = KR + e / 7, coordinate i = e % 7) at columns 2e, 2e + 1, moved as
// three 16-column accesses and one of 8.  f(m, i, v) sees compile-time m and i after unrolling.
template <int E0, int NE, class F>
__device__ __forceinline__ void tm_elems(const float* v, F&& f) {
#pragma unroll
  for (int q = 0; q < NE; ++q)
    f(KR + (E0 + q) / J, (E0 + q) % J, make_float2(v[2 * q], v[2 * q + 1]));
}
template <class F>
__device__ __forceinline__ void for_tm_half(uint32_t tp, F&& f) {
  float v[16];
  tm::ld16_wait<0>(tp, v);
  tm_elems<0, 8>(v, f);
  tm::ld16_wait<16>(tp, v);
  tm_elems<8, 8>(v, f);
  tm::ld16_wait<32>(tp, v);
  tm_elems<16, 8>(v, f);
  tm::ld8_wait<48>(tp, v);
  tm_elems<24, 4>(v, f);
}
// gen(m, i) -> float2 written to the lane's TMEM half (no wait: the caller waits for the stores)
template <int E0, int NE, class Gen>
__device__ __forceinline__ void tm_fill(float* v, Gen&& gen) {
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    const float2 a = gen(KR + (E0 + q) / J, (E0 + q) % J);
    v[2 * q] = a.x;
    v[2 * q + 1] = a.y;
  }
}
template <class Gen>
__device__ __forceinline__ void store_tm_half(uint32_t tp, Gen&& gen) {
  float v[16];
  tm_fill<0, 8>(v, gen);
  tm::st16<0>(tp, v);
  tm_fill<8, 8>(v, gen);
  tm::st16<16>(tp, v);
  tm_fill<16, 8>(v, gen);
  tm::st16<32>(tp, v);
  tm_fill<24, 4>(v, gen);
  tm::st8<48>(tp, v);
}
// f(m, i, old) -> new value, in place
template <int E0, int NE, class F>
__device__ __forceinline__ void tm_map_elems(float* v, F&& f) {
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    const float2 a = f(KR + (E0 + q) / J, (E0 + q) % J, make_float2(v[2 * q], v[2 * q + 1]));
    v[2 * q] = a.x;
    v[2 * q + 1] = a.y;
  }
}
template <class F>
__device__ __forceinline__ void map_tm_half(uint32_t tp, F&& f) {
  float v[16];
  tm::ld16_wait<0>(tp, v);
  tm_map_elems<0, 8>(v, f);
  tm::st16<0>(tp, v);
  tm::ld16_wait<16>(tp, v);
  tm_map_elems<8, 8>(v, f);
  tm::st16<16>(tp, v);
  tm::ld16_wait<32>(tp, v);
  tm_map_elems<16, 8>(v, f);
  tm::st16<32>(tp, v);
  tm::ld8_wait<48>(tp, v);
  tm_map_elems<24, 4>(v, f);
  tm::st8<48>(tp, v);
}

// Slot layout inside a group (XOR-relative): register slot q (pair q / 2, side q & 1) of lane g
// holds the data of the group's point slot q ^ g (of either half), so the recursive-halving
// reduce-scatter keeps and sends STATIC registers (no per-lane selects) and lane g ends up
// with the sum of point slot g in register slot 0; the all-gather is shfl_xor by q.
// First of the two points (sides x, y) of register pair m (0..KP-1) on lane g of group gid; the
// second is k0 ^ 1.
__device__ __forceinline__ int pair_point0(int m, int g, int gid) {
  const int s0 = (2 * (m % KR)) ^ g;  // point slot of side x
  return 2 * (((m / KR) * KR + (s0 >> 1)) * NG + gid) + (s0 & 1);
}
__device__ __forceinline__ float2 shfl_xor2(float2 v, int mask) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}
// Reduce-scatter of 8 per-point values (4 float2 register pairs) across the 8 lanes of a group:
// lane g returns the sum for point slot g.  Fixed tree (bitwise deterministic).
__device__ __forceinline__ float group_rs8(const float2* v) {
  float2 a0 = __fadd2_rn(v[0], shfl_xor2(v[2], 4));
  const float2 a1 = __fadd2_rn(v[1], shfl_xor2(v[3], 4));
  a0 = __fadd2_rn(a0, shfl_xor2(a1, 2));
  return a0.x + __shfl_xor_sync(0xffffffffu, a0.y, 1);
}
// All-gather of one value per lane of the group into 4 float2 register pairs: register slot q
// receives the value of point slot q ^ g, owned by lane g ^ q.
__device__ __forceinline__ void group_ag8(float mine, float2* out) {
  out[0].x = mine;
  out[0].y = __shfl_xor_sync(0xffffffffu, mine, 1);
#pragma unroll
  for (int m = 1; m < G / 2; ++m) {
    out[m].x = __shfl_xor_sync(0xffffffffu, mine, 2 * m);
    out[m].y = __shfl_xor_sync(0xffffffffu, mine, 2 * m + 1);
  }
}
// Sum the 7 per-lane column partials over the 4 groups of the warp (lanes of group 0 then
// hold the warp totals of their coordinates) and write them, with v7 in column 8 g + 7, as the
// warp's partial row (two 16-byte stores per lane of group 0).
// GROUP_ROWS (the IRLS kernel): no fold - `row` is the lane's GROUP row and every lane stores its
// 7 column partials and v7; the consensus warp then sums NG rows in a tree whose first two levels
// are exactly the fold's (bitwise the same sums; 17.26 vs 17.94 ms on config 1.  The ADMM kernel
// keeps the fold: with group rows it measured 2.7 % slower, its consensus chain being longer).
template <bool GROUP_ROWS = false>
__device__ __forceinline__ void fold_store(float (&v)[J], float v7, float* row, int lane) {
  if constexpr (GROUP_ROWS) {
    float4* d = reinterpret_cast<float4*>(row + 8 * (lane & (G - 1)));
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v7);
  } else {
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
}
// Column pair (2 lane, 2 lane + 1) summed over the NR partial rows in a fixed tree.
template <int NR = WARPS>
__device__ __forceinline__ float2 rows_sum(const float* red, int lane) {
  float2 r[NR];
#pragma unroll
  for (int w = 0; w < NR; ++w) r[w] = reinterpret_cast<const float2*>(red + w * RS)[lane];
#pragma unroll
  for (int span = 1; span < NR; span <<= 1)
#pragma unroll
    for (int w = 0; w + span < NR; w += 2 * span) r[w] = __fadd2_rn(r[w], r[w + span]);
  return r[0];
}
// columns 2 l, 2 l + 1 of a published row: the consensus lane l's pair.  SKEW (ADMM): columns
// 32..63 4 floats on; the IRLS kernel keeps the plain row.
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
// next write of `scal` happens after the next problem's barriers.
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

// One problem's points and weights from the shared-memory stage: pairs 0..KR-1 into registers,
// pairs KR.. into this lane's TMEM columns (raw), with the fused input validation (types.hpp:58-68, the
// checks validate_points_dev runs as a separate pass) and the all-points-equal test.  Padding
// slots (k >= n, coordinates >= 49) hold finite 0.  Returns (any element != point 0's).
struct Loaded {
  bool bad_pt, neq;
};
__device__ __forceinline__ Loaded load_problem(const float* __restrict__ src,
                                               const float* __restrict__ wsrc, int n, int gid,
                                               int g, bool is_pts, float2 (&A)[KR][J],
                                               float2 (&wq)[KP], uint32_t tp) {
  const bool greal = is_pts && g < 7;  // lane g = 7 of a group: padding coordinates 49..55
  const float* const col = src + 7 * g;
  float r0[J];
#pragma unroll
  for (int i = 0; i < J; ++i) r0[i] = greal ? col[i] : 0.0f;
  bool bad = false, neq = false;
  auto fetch = [&](int m, int i) {
    const int k0 = pair_point0(m, g, gid), k1 = k0 ^ 1;
    const bool h0 = greal && k0 < n, h1 = greal && k1 < n;
    const float v0 = h0 ? col[k0 * D + i] : r0[i];
    const float v1 = h1 ? col[k1 * D + i] : r0[i];
    neq |= (v0 != r0[i]) | (v1 != r0[i]);
    bad |= !isfinite(v0) | !isfinite(v1);
    return make_float2(h0 ? v0 : 0.0f, h1 ? v1 : 0.0f);
  };
  if (is_pts) {
    store_tm_half(tp, fetch);
    tm::wait_st();
  }
#pragma unroll
  for (int m = 0; m < KR; ++m)
#pragma unroll
    for (int i = 0; i < J; ++i) A[m][i] = fetch(m, i);
#pragma unroll
  for (int m = 0; m < KP; ++m) {
    const int k0 = pair_point0(m, g, gid), k1 = k0 ^ 1;
    wq[m] = make_float2(is_pts && k0 < n ? wsrc[k0] : 0.0f, is_pts && k1 < n ? wsrc[k1] : 0.0f);
  }
  return Loaded{bad, neq};
}
// lowest failing (problem << 2 | code) wins; code 1 coordinates, 2 weights, 3 no positive
// weight - the reference's order within a problem.  One barrier per problem.
__device__ __forceinline__ void check_problem(bool bad_pt, const float2 (&wq)[KP], int64_t b,
                                              unsigned long long* invalid) {
  if (invalid == nullptr) return;  // uniform
  bool bad_w = false, pos = false;
#pragma unroll
  for (int m = 0; m < KP; ++m) {
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
template <bool GROUP_ROWS = false>
__device__ __forceinline__ void weighted_sum_rows(const float2 (&A)[KR][J], uint32_t tp,
                                                  const float2 (&wq)[KP], float* myrow,
                                                  bool is_pts, int lane) {
  if (is_pts) {
    float2 acc[J];
#pragma unroll
    for (int i = 0; i < J; ++i) acc[i] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int m = 0; m < KR; ++m)
#pragma unroll
      for (int i = 0; i < J; ++i) acc[i] = __ffma2_rn(wq[m], A[m][i], acc[i]);
    for_tm_half(tp, [&](int m, int i, float2 a) { acc[i] = __ffma2_rn(wq[m], a, acc[i]); });
    float v[J];
#pragma unroll
    for (int i = 0; i < J; ++i) v[i] = acc[i].x + acc[i].y;
    float ws = 0.0f;  // weights of this lane's group (same in its 8 lanes), then of the warp
#pragma unroll
    for (int m = 0; m < KP; ++m) ws += wq[m].x + wq[m].y;
    if constexpr (GROUP_ROWS) {
      fold_store<true>(v, (lane & (G - 1)) == 0 ? ws : 0.0f, myrow, lane);
    } else {
      ws += __shfl_xor_sync(0xffffffffu, ws, 8);
      ws += __shfl_xor_sync(0xffffffffu, ws, 16);
      fold_store(v, lane == 0 ? ws : 0.0f, myrow, lane);
    }
  }
  __syncthreads();
}

// warp (or, GROUP_ROWS, 8-lane group) sums of four per-lane values (x0..x3) onto lanes
// r = lane & 3 (value x_r)
template <bool GROUP_ROWS = false>
__device__ __forceinline__ float quad_sums(float x0, float x1, float x2, float x3, int lane) {
  const bool u2 = (lane & 2) != 0, u1 = (lane & 1) != 0;
  const float y0 = (u2 ? x2 : x0) + __shfl_xor_sync(0xffffffffu, u2 ? x0 : x2, 2);
  const float y1 = (u2 ? x3 : x1) + __shfl_xor_sync(0xffffffffu, u2 ? x1 : x3, 2);
  float hs = (u1 ? y1 : y0) + __shfl_xor_sync(0xffffffffu, u1 ? y0 : y1, 1);
#pragma unroll
  for (int o = 4; o < (GROUP_ROWS ? G : 32); o <<= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
  return hs;
}

}  // namespace blr

using namespace blr;

__global__ void __launch_bounds__(ALL, 2)
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
  // TMEM: the second half of every lane's points (128 columns per CTA, two CTAs per SM)
  const uint32_t tbase = tm::alloc_cta<TM_COLS>(reinterpret_cast<uint32_t*>(smem + SM_TB), warp);
  const uint32_t tp = tm::warp_addr(tbase, warp, (warp >> 2) * TM_WCOLS);
  float* const myrow = red + (is_pts ? warp : 0) * RS;
  const bool greal = is_pts && g < 7;
  // this lane's two point slots: point slot g of each half (its register slot 0)
  int k_me[2];
  bool real_me[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    k_me[h] = pair_point0(KR * h, g, gid);  // register slot 0 = point slot g
    real_me[h] = is_pts && k_me[h] < n;
  }
  // consensus (warp CW): lane l finishes columns 2l, 2l+1 = coordinates cj, cj + 1
  const int cgrp = lane >> 2, cidx = 2 * (lane & 3);
  const int cj = 7 * cgrp + cidx;
  const bool cv0 = cgrp < 7, cv1 = cgrp < 7 && (lane & 3) != 3;
  const float inv_mu = 1.0f / mu;
  const float inv_n = 1.0f / static_cast<float>(n);
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
    // ---- this problem's points (raw) into registers / TMEM, weights, all-equal test
    const float* const src = stage + stage_shift(points + b * nd);
    const float* const wsrc = wst + stage_shift(weights + b * n);
    float2 A[KR][J];
    float2 wq[KP];
    const Loaded ld = load_problem(src, wsrc, n, gid, g, is_pts, A, wq, tp);
    float w_me[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) w_me[h] = real_me[h] ? wsrc[k_me[h]] : 0.0f;
    check_problem(ld.bad_pt, wq, b, invalid);
    const bool static_eq = !__syncthreads_or(ld.neq);  // every thread is done with the stage
    if (b + gridDim.x < batch) {  // the next problem streams in during this one's sweeps
      stage_copy(stage, points + (b + gridDim.x) * nd, nd);
      stage_copy(wst, weights + (b + gridDim.x) * n, n);
    }
    cp_commit();
    // exact stop possible (the p-form kernel decides it structurally), or the small-mu regime
    if (static_eq || all_mode) {
      if (tid == 0) ho_list[atomicAdd(ho_count, 1)] = static_cast<int>(b);
      continue;
    }

    // ---- z_0 = m: z_init, or the weighted mean points * (w / sum w) (admm.hpp:40, types.hpp:73)
    float m0 = 0.0f, m1 = 0.0f;  // consensus warp: m at coordinates cj, cj + 1
    if (z_init == nullptr) weighted_sum_rows(A, tp, wq, myrow, is_pts, lane);
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
    // centre the points on m; ||a~||^2 of this lane's two points
    float a2[2];
    {
      float mc[J];
      load_coords(mb, g, mc);
      float2 nq[KP];
#pragma unroll
      for (int m = 0; m < KP; ++m) nq[m] = make_float2(0.0f, 0.0f);
      auto centre = [&](int m, int i, float2 a) {
        const int k0 = pair_point0(m, g, gid);
        const float2 c = make_float2(greal && k0 < n ? a.x - mc[i] : 0.0f,
                                     greal && (k0 ^ 1) < n ? a.y - mc[i] : 0.0f);
        nq[m] = __ffma2_rn(c, c, nq[m]);
        return c;
      };
#pragma unroll
      for (int m = 0; m < KR; ++m)
#pragma unroll
        for (int i = 0; i < J; ++i) A[m][i] = centre(m, i, A[m][i]);
      if (is_pts) {
        map_tm_half(tp, centre);
        tm::wait_st();
      }
      a2[0] = group_rs8(nq);
      a2[1] = group_rs8(nq + KR);
    }
    // per-point state (own slots): p_1 = z_0 - a = -a~ (u = 0, admm.hpp:41)
    float H[2], K[2], ga[2], al0[2], al1[2], al2[2], al3[2], lam[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      H[h] = a2[h];
      K[h] = -a2[h];
      ga[h] = al0[h] = al1[h] = al2[h] = al3[h] = 0.0f;
      lam[h] = inv_mu * w_me[h];
    }
    // consensus state (warp CW): z, history ring c~_{t-r} (r = 0..3) and its norms
    float z0 = m0, z1 = m1;
    float h0[R], h1[R], nr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) h0[r] = h1[r] = nr[r] = 0.0f;
    bool bad = false;  // consensus warp: non-finite iterate
    float hov = 0.0f;  // point lanes: running maximum of the hand-off tests

    for (int t = 1; t <= T; ++t) {
      if (is_pts) {
        // (1) D_k = <a~_k, c~_t>
        // c~_t is published by the consensus warp before its Gram row (named barriers): the dot
        // products overlap the Gram reduction
        if (t > 1) bar_sync(BAR_C);
        float Dk[2];
        {
          float cv[J];
          load_coords(cb, g, cv);
          float2 dq[KP];
#pragma unroll
          for (int m = 0; m < KP; ++m) dq[m] = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < J; ++i)
#pragma unroll
            for (int m = 0; m < KR; ++m) dq[m] = __ffma2_rn(A[m][i], f2(cv[i]), dq[m]);
          for_tm_half(tp, [&](int m, int i, float2 a) { dq[m] = __ffma2_rn(a, f2(cv[i]), dq[m]); });
          Dk[0] = group_rs8(dq);
          Dk[1] = group_rs8(dq + KR);
        }
        // (2) scalar update of this lane's points
        if (t > 1) {
          pin[tid] = Dk[0] + Dk[1];  // the dot products and their reduction run before the wait
          bar_sync(BAR_GRAM);
        }
        const float4 gq4 = reinterpret_cast<const float4*>(gr)[0];
        const float2 gq2 = reinterpret_cast<const float2*>(gr)[2];
        const float Gnn = gq2.x, nrR = gq2.y;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float X = fmaf(al0[h], gq4.x, fmaf(al1[h], gq4.y, fmaf(al2[h], gq4.z, al3[h] * gq4.w)));
          const float gp1 = ga[h] + 1.0f;
          const float HG = H[h] + Gnn;
          const float N = fmaf(2.0f, fmaf(-gp1, Dk[h], X), HG);
          const float Nc = fmaxf(N, 0.0f);
          const float s = lam[h] != 0.0f ? fminf(1.0f, lam[h] * rsq(Nc)) : 0.0f;
          const float Bk = K[h] + Dk[h];
          const float ev = s * al3[h];
          // hand-off tests as one running maximum (> 0: hand off): a dropped ring term above
          // rounding, or a cancelling N (zero-weight points included: a spurious hand-off only
          // costs time)
          hov = fmaxf(hov, fmaxf(fmaf(ev * ev, nrR, -kThr2 * Nc), fmaf(kCancel, HG, -N)));
          // N unclamped: a non-finite N (or D) makes H non-finite for good, tested after the
          // last sweep instead of every sweep
          H[h] = fmaf(s, fmaf(s, N, -2.0f * Bk), a2[h]);
          K[h] = fmaf(s, Bk, -a2[h]);
          ga[h] = s * gp1;
          al3[h] = s * al2[h];
          al2[h] = s * al1[h];
          al1[h] = s * al0[h];
          al0[h] = s;
        }
        // (3) sum_k ga'_k a~_k per coordinate; history sums sum_k al'_r (onto lanes r = 0..3)
        float v[J];
        {
          float2 acc[J];
#pragma unroll
          for (int i = 0; i < J; ++i) acc[i] = make_float2(0.0f, 0.0f);
          float2 gq[KP];
          group_ag8(ga[0], gq);
          group_ag8(ga[1], gq + KR);
#pragma unroll
          for (int m = 0; m < KR; ++m)
#pragma unroll
            for (int i = 0; i < J; ++i) acc[i] = __ffma2_rn(gq[m], A[m][i], acc[i]);
          for_tm_half(tp, [&](int m, int i, float2 a) { acc[i] = __ffma2_rn(gq[m], a, acc[i]); });
#pragma unroll
          for (int i = 0; i < J; ++i) v[i] = acc[i].x + acc[i].y;
        }
        const float hs = quad_sums(al0[0] + al0[1], al1[0] + al1[1], al2[0] + al2[1],
                                   al3[0] + al3[1], lane);
        fold_store(v, lane < 4 ? hs : 0.0f, myrow, lane);
        __syncthreads();
      } else {
        __syncthreads();
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
      }
    }

    // ---- hand-off or outputs
    if (__syncthreads_or(bad || hov > 0.0f || !isfinite(H[0]) || !isfinite(H[1]))) {
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
      auto dist = [&](int m, int i, float2 a) {
        const float2 e = __fadd2_rn(f2(zc[i]), make_float2(-a.x, -a.y));
        const float2 em = 7 * g + i < D ? e : make_float2(0.0f, 0.0f);
        dq[m] = __ffma2_rn(em, em, dq[m]);
      };
#pragma unroll
      for (int m = 0; m < KR; ++m)
#pragma unroll
        for (int i = 0; i < J; ++i) dist(m, i, A[m][i]);
      if (is_pts) for_tm_half(tp, dist);
      const float d0 = group_rs8(dq), d1 = group_rs8(dq + KR);
      const float mine = (real_me[0] ? w_me[0] * sqrtf(d0) : 0.0f) +
                         (real_me[1] ? w_me[1] * sqrtf(d1) : 0.0f);
      const float obj = block_sum0(mine, scal, warp, lane);
      if (tid == 0) {
        obj_out[b] = obj;
        if (!isfinite(obj)) ho_list[atomicAdd(ho_count, 1)] = static_cast<int>(b);
      }
    }
  }
  cp_wait_all();
  tm::dealloc_cta<TM_COLS>(tbase, warp);
}

// ---------------------------------------------------------------------------------------
// Batched IRLS (proj/include/nlem/irls.hpp:21-68), d = 49, 1 <= n <= 448: the same layout
// (half of the points in registers, half in tensor memory, two problems per SM) and consensus
// warp, direct differences (exact near coincident points, where epsilon matters).  Pass p
// evaluates at x_p: per point D = ||x_p - a_k||^2 (FADD2 + FFMA2), root = sqrt(D + eps), beta =
// w / root, the surrogate term w root (costs.hpp:24-33) and the cost term w sqrt(D)
// (costs.hpp:13-20, the objective output at the final x); the point warps reduce sum beta a,
// sum beta, the surrogate and the cost; the consensus warp applies the stop rule (irls.hpp:58)
// and forms x_{p+1} = sum beta a / sum beta.  Failures are recorded as the generic kernel does
// (iteration and kind of irls.hpp:39, :50, :52, :65-66).
// ---------------------------------------------------------------------------------------
namespace blr {
// shared memory of the IRLS kernel (floats): stage and weights as above, then one partial row
// per 8-lane group, x of the coming pass, the control word and the TMEM base
constexpr int SI_CB = SM_RED + NG * RS;
constexpr int SI_CTL = SI_CB + RSK;
constexpr int SI_TB = SI_CTL + 4;
constexpr int SI_TOTAL = SI_TB + 4;
constexpr size_t SMEM_BYTES_IRLS = size_t(SI_TOTAL) * sizeof(float);
static_assert(SI_CB % 4 == 0 && 2 * (SMEM_BYTES_IRLS + 1024) <= 233472, "two IRLS CTAs per SM");
}  // namespace blr

__global__ void __launch_bounds__(ALL, 2)
irls_batched_reg(const float* __restrict__ points, const float* __restrict__ weights,
                 int64_t batch, int n, const float* __restrict__ x_init, float eps, int T,
                 float tol, float* x_out, float* obj_out, int* iters_out, float* tr_obj,
                 FailureSlot* fail, unsigned long long* invalid) {
  extern __shared__ __align__(16) float smem[];
  float* const stage = smem + SM_STAGE;
  float* const wst = smem + SM_WST;
  float* const red = smem + SM_RED;  // [NG][RS]: one partial row per 8-lane group
  float* const cb = smem + SI_CB;    // x of the coming pass
  int* const ctl = reinterpret_cast<int*>(smem + SI_CTL);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int lane = tid & 31;
  const int g = lane & (G - 1);
  const int gid = warp * GPW + (lane >> 3);
  const bool is_pts = warp < WARPS;
  // TMEM: the second half of every lane's points (128 columns per CTA, two CTAs per SM)
  const uint32_t tbase = tm::alloc_cta<TM_COLS>(reinterpret_cast<uint32_t*>(smem + SI_TB), warp);
  const uint32_t tp = tm::warp_addr(tbase, warp, (warp >> 2) * TM_WCOLS);
  float* const myrow = red + (is_pts ? gid : 0) * RS;
  int k_me[2];
  bool real_me[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    k_me[h] = pair_point0(KR * h, g, gid);  // register slot 0 = point slot g
    real_me[h] = is_pts && k_me[h] < n;
  }
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
    const float* const src = stage + stage_shift(points + b * nd);
    const float* const wsrc = wst + stage_shift(weights + b * n);
    float2 A[KR][J];
    float2 wq[KP];
    const Loaded ld = load_problem(src, wsrc, n, gid, g, is_pts, A, wq, tp);
    float w_me[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) w_me[h] = real_me[h] ? wsrc[k_me[h]] : 0.0f;
    check_problem(ld.bad_pt, wq, b, invalid);
    __syncthreads();  // every thread is done with the stage
    if (b + gridDim.x < batch) {  // the next problem streams in during this one's passes
      stage_copy(stage, points + (b + gridDim.x) * nd, nd);
      stage_copy(wst, weights + (b + gridDim.x) * n, n);
    }
    cp_commit();

    // ---- x_0: x_init, or the weighted mean points * (w / sum w) (irls.hpp:32, types.hpp:73)
    if (x_init == nullptr) weighted_sum_rows<true>(A, tp, wq, myrow, is_pts, lane);
    float x0 = 0.0f, x1 = 0.0f;  // consensus warp: x of the current pass at cj, cj + 1
    if (warp == CW) {
      if (x_init != nullptr) {
        x0 = cv0 ? x_init[b * D + cj] : 0.0f;
        x1 = cv1 ? x_init[b * D + cj + 1] : 0.0f;
      } else {
        const float2 s = rows_sum<NG>(red, lane);
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
        // no mask for the padding coordinates of lanes g = 7: their points are 0 and x's
        // padding columns are written as exact zeros (cv0 / cv1), so e = 0 there
        auto dist = [&](int m, int i, float2 a) {
          const float2 e = __fadd2_rn(f2(xc[i]), make_float2(-a.x, -a.y));
          dq[m] = __ffma2_rn(e, e, dq[m]);
        };
#pragma unroll
        for (int i = 0; i < J; ++i)
#pragma unroll
          for (int m = 0; m < KR; ++m) dist(m, i, A[m][i]);
        for_tm_half(tp, dist);
        float d2[2] = {group_rs8(dq), group_rs8(dq + KR)};
        // irls.hpp:45-46 and costs.hpp:24-33 / :13-20 with one hardware reciprocal square root
        // per point each (rsqrt.approx: ~2 ulp, against an FP64 reference)
        float beta[2], sur = 0.0f, cost = 0.0f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float s2 = d2[h] + eps;
          const float ri = rsq(s2);
          beta[h] = real_me[h] ? w_me[h] * ri : 0.0f;
          sur += real_me[h] ? w_me[h] * (s2 * ri) : 0.0f;
          cost += real_me[h] && d2[h] > 0.0f ? w_me[h] * (d2[h] * rsq(d2[h])) : 0.0f;
        }
        float v[J];
        {
          float2 acc[J];
#pragma unroll
          for (int i = 0; i < J; ++i) acc[i] = make_float2(0.0f, 0.0f);
          float2 bq[KP];
          group_ag8(beta[0], bq);
          group_ag8(beta[1], bq + KR);
#pragma unroll
          for (int m = 0; m < KR; ++m)
#pragma unroll
            for (int i = 0; i < J; ++i) acc[i] = __ffma2_rn(bq[m], A[m][i], acc[i]);
          for_tm_half(tp, [&](int m, int i, float2 a) { acc[i] = __ffma2_rn(bq[m], a, acc[i]); });
#pragma unroll
          for (int i = 0; i < J; ++i) v[i] = acc[i].x + acc[i].y;
        }
        // warp sums of (beta, surrogate, cost, 0) onto lanes r = lane & 3
        const float hs = quad_sums<true>(beta[0] + beta[1], sur, cost, 0.0f, lane);
        fold_store<true>(v, g < 4 ? hs : 0.0f, myrow, lane);
      }
      __syncthreads();
      if (warp == CW) {
        const float2 S = rows_sum<NG>(red, lane);
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
  tm::dealloc_cta<TM_COLS>(tbase, warp);
}

// persistent grid: two CTAs per SM (registers: 2 x 256 threads x 128; shared memory below)
constexpr int kCtasPerSm = 2;
constexpr int kCarveoutPct =
    static_cast<int>((kCtasPerSm * (SMEM_BYTES + 1024) * 100 + 233471) / 233472) + 2;

bool irls_reg_supported(const IrlsLaunch& L) {
  const char* force = std::getenv("NLEM_BATCHED");  // =fast: the generic IRLS kernel (A/B, tests)
  if (force != nullptr && std::string(force) != "lr") return false;
  return L.d == D && L.n >= 1 && L.n <= NCAP && L.batch < (int64_t(1) << 31) &&
         static_cast<int64_t>(L.n) * D < (int64_t(1) << 31) / 4;
}

cudaError_t launch_irls_reg(const IrlsLaunch& L, cudaStream_t stream) {
  auto kfn = irls_batched_reg;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES_IRLS));
  if (e != cudaSuccess) return e;
  // shared-memory carve-out for kCtasPerSm resident CTAs (the rest of the 256 KB stays L1)
  constexpr int carve =
      static_cast<int>((kCtasPerSm * (SMEM_BYTES_IRLS + 1024) * 100 + 233471) / 233472) + 2;
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(L.batch, int64_t(kCtasPerSm) * device_caps().sms));
  kfn<<<static_cast<unsigned>(grid), ALL, SMEM_BYTES_IRLS, stream>>>(
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
  // shared-memory carve-out for kCtasPerSm resident CTAs (the rest of the 256 KB stays L1)
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, kCarveoutPct);
  if (e != cudaSuccess) return e;
  if (probe != nullptr && L.max_iter > R) {
    const int pn = static_cast<int>(std::min<int64_t>(L.batch, kProbe));
    small_mu_probe_kernel<<<pn, 256, 0, stream>>>(L.points, L.weights, L.batch, L.n, L.z_init,
                                                  L.mu, pn, probe);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else {
    probe = nullptr;
  }
  if (std::getenv("NLEM_LR_STATS") != nullptr) {  // diagnostics only
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, ALL, SMEM_BYTES);
    std::fprintf(stderr, "admm_batched_lr: %d resident CTAs per SM\n", occ);
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(L.batch, int64_t(kCtasPerSm) * device_caps().sms));
  kfn<<<static_cast<unsigned>(grid), ALL, SMEM_BYTES, stream>>>(
      L.points, L.weights, L.batch, L.n, L.z_init, L.box, L.mu, L.max_iter, L.z_out, L.obj_out,
      L.iters_out, ho_list, ho_count, L.invalid, probe);
  return cudaGetLastError();
}

}  // namespace nlemk
