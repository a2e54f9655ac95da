// Low-rank ("Gram-form") NLEM / EM-ADMM kernel for k = 7, S <= 21 (configs 2, 3, 4; windows
// smaller than 21 run masked inside the 21 x 21 grid); also the IRLS comparator and the NlmOnly
// solver / nlm_denoise baseline in the same mapping.
//
// Algebra (p-form of admm.hpp:49-78).  With p_k = z - y_k/mu - a_k and
// s_k = min(1, lambda_k / ||p_k||), one sweep is
//     z' = P_C(z - (1/n) sum_k s_k p_k),   p_k' = s_k p_k + c' - a_k,   c' = 2 z' - z.
// Unrolling the recursion, s_k p_k is always a combination of the point a_k and the shared
// history c_1, c_2, ... of consensus vectors:  s p = sum_r al_r c~_{t-r} - ga a~_k, where
// everything is centred on m = a_self (the coefficients sum to zero, so the centring is exact
// in real arithmetic).  The history coefficients are products of prox scales (s << 1 in the
// configs: lambda = w/mu <= 1 against ||p|| ~ 100), so only the last R = 4 of them are ever
// significant; an older one is dropped only when its vector is below 2^-22 ||p||, i.e. under
// FP32 rounding of p itself.  A pixel whose ring would drop a significant term is handed to the
// exact p-form tile kernel (kernels_nlem_tile.cu) through a device-side pixel list.
//
// Per point the state is 8 scalars (H = ||s p - a~||^2, K = <s p - a~, a~>, ga, ||a~||^2, al_0..3)
// instead of the d = 49 floats of the p-form, and a sweep costs one dot product
// D_k = <a~_k, c~> and one weighted patch sum sum_k ga_k a~_k (two FMAs per element) plus a few
// scalar ops per point:
//     N = H + 2 (sum_r al_r <c~_{t-1-r}, c~_t> - (ga + 1) D) + ||c~_t||^2      (= ||p_k||^2)
//     s = min(1, lambda rsqrt(N));  B = K + D;  H' = s (s N - 2 B) + ||a~||^2;  K' = s B - ||a~||^2
//     ga' = s (ga + 1);  al' = (s, s al_0, s al_1, s al_2)
//     g = sum_k s p_k = sum_r (sum_k al'_r) c~_{t-r} - sum_k ga'_k a~_k.
// The algorithmic FLOP count (12 d per point and sweep) is unchanged.
//
// Mapping (B200): ONE PIXEL PER WARP, 16 independent pixel-warps per SM - no CTA barrier on
// the sweep path, so one warp's reduction latency is hidden by the other fifteen's FMAs.
//  * lane l owns two vertical segments of 7 grid points (63 segments = 441 points) that read
//    the same relative tile offsets, so the pixel's 27 x 27 tile sits in shared memory as two
//    PAIRED column-major copies ((slot 0, slot 1) float2 per tile row, see the layout below):
//    a paired column (seven 16-byte loads) serves 49 FFMA2 of the dot products, the distances
//    and the patch sums.  The tile streams in with 4-byte cp.async at the end of the previous
//    pixel (its latency is not exposed: other warps compute);
//  * the per-point state (8 x 32-bit) lives in TENSOR MEMORY: 14 points x 8 columns + 14
//    lambdas per lane = 128 columns per warp, 16 warps = all 512 columns x 128 lanes of the SM,
//    moved with tcgen05.ld x16 / st x2 - registers stay free for the FMA working set;
//  * the 54 per-lane partials (49 coordinates, sum ga, 4 history sums) are reduced with a
//    shared-memory transpose (fixed tree: bitwise deterministic), the 49 consensus coordinates
//    are finished by their owner lanes, which keep z, m and the c~ history in shared memory;
//    the Gram row <c~_{t-r}, c~_{t+1}> is a 6-value butterfly all-reduce kept in registers;
//  * the point state of pair i + 1 is requested from TMEM (tcgen05.ld) before the arithmetic of
//    pair i, the previous sweep's stores are waited for only there.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "launch.h"
#include "tmem.cuh"

namespace nlemk {

namespace lr {

constexpr int KS = 7, SW = 21, HS = SW / 2;
constexpr int TH = SW + KS - 1;  // 27
// Tile layout: two PAIRED column-major copies.  A lane's two segments always read the same
// relative (row, column) offsets, so their tile values are stored interleaved as (slot 0, slot 1)
// float2 pairs and every correlation step is one FFMA2 on a pair:
//  * copy A (lanes 0..20: segments (x, grid rows 0..6) and (x, rows 7..13)):
//    A[x][r] = (T[r][x], T[r + 7][x]), r = 0..12, x = 0..26;
//  * copy B (lanes 21..31: segments (x, rows 14..20) and (x + 11, rows 14..20), x = 0..10; lane
//    31's second segment does not exist): B[x][r] = (T[14 + r][x], T[14 + r][x + 11]), x = 0..16.
// A column is 14 pairs (pair 13 = 0 padding) = seven 16-byte loads; stride PCS = 28 floats (odd
// number of 16-byte quads: 8 consecutive columns hit 8 distinct bank quads) and PB = PA + 12
// mod 32 keeps the LDS.128 phase that straddles the two copies (lanes 16..23) conflict-free.
constexpr int PCS = 28;
constexpr int PA = 0, PB = 780;
constexpr int BCOLS = 17;
constexpr int TILE = PB + BCOLS * PCS;  // 1256 floats
static_assert((PB - PA) % 32 == 12 && PB >= TH * PCS, "copy B placement");
#ifndef NLEM_LR_WARPS
#define NLEM_LR_WARPS 16
#endif
constexpr int WARPS = NLEM_LR_WARPS;  // pixel-warps per CTA (1 CTA per SM)
constexpr int SEGL = 7;  // points per segment
// History ring length.  4 in the production build (16 pixel-warps per SM); the second
// translation unit kernels_nlem_lr_r12.cu compiles this file with NLEM_LR_R = 12 and 8 warps
// for the small-mu regime (prox scales of 1: no history term decays, so the ring must hold all
// T <= 12 sweeps; twice the tensor-memory columns per pixel, hence half the warps).
#ifndef NLEM_LR_R
#define NLEM_LR_R 4
#endif
constexpr int R = NLEM_LR_R;
constexpr int NF = 4 + R;       // state fields per point in TMEM: H, K, ga, ||a~||^2, al_0..R-1
constexpr int PC = 2 * NF;      // TMEM columns of one point pair (16 or 32)
constexpr int TCW = R == 4 ? 128 : 256;  // TMEM columns per pixel-warp
static_assert(PC == 16 || PC == 32, "point pairs move as one or two x16 accesses");
static_assert(SEGL * PC + 16 <= TCW && (WARPS / 4) * TCW <= 512 && WARPS % 4 == 0, "TMEM budget");
#ifndef NLEM_LR_NAME
#define NLEM_LR_NAME nlem_pixels_lr
#endif
// unroll factors of the correlation loops over patch columns (A/B build variants)
#ifndef NLEM_LR_UD
#define NLEM_LR_UD 7  // A/B on the paired layout: 7 (unrolled) 32.23 vs 1 (rolled) 32.00 Mpix/s
#endif
#ifndef NLEM_LR_UG
#define NLEM_LR_UG 1
#endif
#define LR_PRAGMA(x) _Pragma(#x)
#define LR_UNROLL(n) LR_PRAGMA(unroll n)
constexpr int RED_STR = 36;
constexpr int CB_STR = 8;
// per-warp shared memory (floats)
constexpr int W_RED = TILE;  // single tile buffer
constexpr int W_CB = W_RED + 32 * RED_STR;
constexpr int W_OWN = W_CB + KS * CB_STR;        // [4 + 2 (R+1)][32] owner scalars
constexpr int W_NR = W_OWN + (4 + 2 * (R + 1)) * 32;  // [R+1] (+pad) ||c~||^2 ring
constexpr int W_TOTAL = W_NR + ((R + 1 + 3) & ~3);
constexpr size_t SMEM_BYTES = size_t(WARPS) * W_TOTAL * sizeof(float) + 16;
constexpr int kProbe = 1024;  // pixels sampled by the small-mu probe launch
constexpr int kCenterLane = 24;  // owner of coordinate D/2 = (3, 3): half A row 3*7+3
constexpr float kThr2 = 1.0f / 17592186044416.0f;  // (2^-22)^2
constexpr float kCancel = 1.0f / 256.0f;  // N below 2^-8 (H + ||c~||^2): the expansion cancels

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// three-input maximum (FMNMX3, sm_100)
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float rsq(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- TMEM (tcgen05) helpers: 32 lanes x N columns of 32-bit per warp access.  Each load is
// issued together with its wait in one asm statement, so no use of the destination registers
// can be scheduled before the data has landed (the loads are asynchronous).
template <int N>
__device__ __forceinline__ void tm_ld_wait(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void tm_ld_wait<8>(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tm_ld_wait<16>(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t taddr, const float* v);
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
template <>
__device__ __forceinline__ void tm_st<16>(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void tm_st1(uint32_t taddr, float v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)) : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, float a, float b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(a)), "r"(__float_as_uint(b)) : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t taddr, float a, float b, float c, float d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)) : "memory");
}
// Base + compile-time column offset (PTX [taddr+imm]): one long-lived base register instead of
// one uniform register per address (those exhausted the uniform register file) or a per-access
// add + R2UR.
template <int OFF>
__device__ __forceinline__ void tm_st1c(uint32_t base, float v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0+%1], {%2};" ::"r"(base), "n"(OFF),
               "r"(__float_as_uint(v))
               : "memory");
}
template <int OFF>
__device__ __forceinline__ void tm_st2c(uint32_t base, float a, float b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+%1], {%2, %3};" ::"r"(base), "n"(OFF),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b))
               : "memory");
}
template <int OFF>
__device__ __forceinline__ void tm_st4c(uint32_t base, float a, float b, float c, float d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0+%1], {%2, %3, %4, %5};" ::"r"(base), "n"(OFF),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)),
               "r"(__float_as_uint(d))
               : "memory");
}
template <int OFF>
__device__ __forceinline__ void tm_ld16c_wait(uint32_t base, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16+%17];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(base), "n"(OFF)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  [&]<int... I>(std::integer_sequence<int, I...>) { (f(std::integral_constant<int, I>{}), ...); }(
      std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float box_clamp(float v, const nlem_box& box) {
  if (!box.bounded) return v;
  const float y = (v < box.lower) ? box.lower : v;
  return (box.upper < y) ? box.upper : y;
}

// Segment geometry: vertical segment (grid column gx, grid rows gy0 .. gy0+6) of a lane's slot.
__device__ __forceinline__ void seg_of(int lane, int slot, int& gx, int& gy0, bool& valid) {
  valid = true;
  if (lane < 21) {
    gx = lane;
    gy0 = slot ? 7 : 0;
  } else {
    gx = lane - 21 + (slot ? 11 : 0);
    gy0 = 14;
    valid = !(slot == 1 && lane == 31);
  }
}

// Forces a float2 into one aligned 64-bit register pair (the FFMA2 operand form), so the
// compiler does not re-pair two scattered 32-bit registers with MOVs at every use.
__device__ __forceinline__ float2 pin_pair(float2 v) {
  unsigned long long b = (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
  asm volatile("" : "+l"(b));
  return make_float2(__uint_as_float(static_cast<unsigned>(b)), __uint_as_float(static_cast<unsigned>(b >> 32)));
}

// tile element (row r, column x) in the paired copies
__device__ __forceinline__ float tile_at(const float* T, int r, int x) {
  if (r < 13) return T[PA + x * PCS + 2 * r];
  if (r < 20) return T[PA + x * PCS + 2 * (r - 7) + 1];
  return x < BCOLS ? T[PB + x * PCS + 2 * (r - 14)] : T[PB + (x - 11) * PCS + 2 * (r - 14) + 1];
}
// the 14 pairs of a paired column: seven 16-byte loads
__device__ __forceinline__ void load_pcol(const float* col, float2 (&v)[14]) {
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const float4 t = reinterpret_cast<const float4*>(col)[q];
    v[2 * q] = make_float2(t.x, t.y);
    v[2 * q + 1] = make_float2(t.z, t.w);
  }
}
// acc[i] += v[i + jy] * c[jy]   (both slots of point i in one FFMA2)
__device__ __forceinline__ void p_dot(float2 (&acc)[7], const float2 (&v)[14], const float (&c)[7]) {
#pragma unroll
  for (int jy = 0; jy < 7; ++jy)
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[i] = __ffma2_rn(v[i + jy], make_float2(c[jy], c[jy]), acc[i]);
}
// acc[i] += (v[i + jy] + nx[jy])^2   (nx = -x)
__device__ __forceinline__ void p_dist(float2 (&acc)[7], const float2 (&v)[14], const float (&nx)[7]) {
#pragma unroll
  for (int jy = 0; jy < 7; ++jy)
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const float2 d = __fadd2_rn(v[i + jy], make_float2(nx[jy], nx[jy]));
      acc[i] = __ffma2_rn(d, d, acc[i]);
    }
}
// g[jy] += u[i] * v[i + jy]   (slot 0 and slot 1 contributions in the two halves of g)
__device__ __forceinline__ void p_gsum(float2 (&g)[7], const float2 (&v)[14], const float2 (&u)[7]) {
#pragma unroll
  for (int i = 0; i < 7; ++i)
#pragma unroll
    for (int jy = 0; jy < 7; ++jy) g[jy] = __ffma2_rn(u[i], v[i + jy], g[jy]);
}
// sum of red[row][0..31] (row stride RED_STR, 16-byte aligned) in a fixed tree order
__device__ __forceinline__ float row_sum(const float* row) {
  float4 q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = reinterpret_cast<const float4*>(row)[i];
  float s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = (q[i].x + q[i].y) + (q[i].z + q[i].w);
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

}  // namespace lr

using namespace lr;

__global__ void __launch_bounds__(WARPS * 32, 1)
NLEM_LR_NAME(const float* __restrict__ pad, int pad_cols, int rows, int cols, int out_row0,
               int plane, NlemDevParams P, float* out, float* frames, int* work_counter,
               int* ovf_list, int* ovf_count, FailureSlot* fail, int probe_n, int* probe_count) {
  // probe_n > 0 (probe launch): only the setup and the small-mu predictor of probe_n pixels
  // spread evenly over the band, counting predicted hand-offs into *probe_count; no outputs.
  // probe_n == 0 with probe_count (main launch): when more than 90 % of the probe pixels
  // would be handed off (the small-mu regime), this launch does no pixel work: up to
  // kLrBigRing sweeps the ring-12 build of this kernel (launched next) takes the band, beyond
  // that *ovf_count = -1 tells the tile kernel to.  The ring-12 launch in turn only works in
  // that regime.  The decision depends on the input only (deterministic).
  if (probe_n == 0 && probe_count != nullptr) {
    const int pt = plane < kProbe ? plane : kProbe;
    const bool small_mu = 10 * *static_cast<volatile int*>(probe_count) > 9 * pt;
#ifdef NLEM_LR_SECONDARY
    if (!small_mu) return;
#else
    if (small_mu) {
      if (P.iters > kLrBigRing && blockIdx.x == 0 && threadIdx.x == 0) *ovf_count = -1;
      return;
    }
#endif
  }
  extern __shared__ __align__(16) float smem[];
  // warp index through a shuffle: the compiler then knows it is warp-uniform (uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  uint32_t* tm_base_slot = reinterpret_cast<uint32_t*>(smem + WARPS * W_TOTAL);
  float* const W = smem + warp * W_TOTAL;
  float* const red = W + W_RED;
  float* const cb = W + W_CB;
  float* const own = W + W_OWN + lane;  // owner scalars, row stride 32 (lane-private column)
  float* const nrs = W + W_NR;          // ||c~||^2 history ring (warp-uniform)

  // ---- TMEM: all 512 columns for this CTA (1 CTA per SM by shared-memory size)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(tm_base_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *tm_base_slot;
  const uint32_t tw = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) +
                      static_cast<uint32_t>((warp >> 2) * TCW);
  // TMEM addresses are formed right before each access (opaque to CSE/hoisting): kept as
  // long-lived uniform registers they exhaust the uniform register file and spill
  auto t_at = [&](uint32_t col) { return tw + col; };
  // column layout per lane: point pair i (slot 0 and slot 1 point i) = 16 columns, field q of
  // slot s at 2 q + s, so one x16 load yields 8 (slot 0, slot 1) register pairs for the paired
  // (FFMA2 / FMUL2 / FADD2) scalar update; lambdas of the 14 points at 112 + 2 i + s
  auto t_pt = [&](int i) { return t_at(static_cast<uint32_t>(i * PC)); };
  auto t_lam = [&]() { return t_at(static_cast<uint32_t>(PC * SEGL)); };

  // lane geometry: segment column offsets in the tile
  int sgx0, sgy00, sgx1, sgy01;
  bool sval0, sval1;
  seg_of(lane, 0, sgx0, sgy00, sval0);
  seg_of(lane, 1, sgx1, sgy01, sval1);
  const int poff = lane < 21 ? PA + lane * PCS : PB + (lane - 21) * PCS;  // paired column base
  // coordinate owners: the reduction runs in two halves (patch columns 0-3 and 4-6); row
  // l of half A is coordinate (l % 7, l / 7), row l of half B is (l % 7, 4 + l / 7)
  const bool own0 = lane < 4 * KS, own1 = lane < 3 * KS;
  const int jy0 = lane % KS, jx0 = lane / KS, jx1 = 4 + lane / KS;

  const float inv_mu = 1.0f / P.mu;
  const int hw = P.search >> 1, wlo = HS - hw;  // masked window for S < 21
  // box as a pair of bounds (infinite when unconstrained): the clamp is two selects
  const float box_lo = P.range.bounded ? P.range.lower : -__int_as_float(0x7f800000);
  const float box_hi = P.range.bounded ? P.range.upper : __int_as_float(0x7f800000);
  const bool nlm_init = P.init_mode == NLEM_INIT_NLM_PATCH;
  const bool irls = P.solver == NLEM_SOLVER_IRLS;
  // NlmOnly (nlem.cpp:26-31, nlm.cpp:31-51): distances and weights as for NLEM, then only the
  // centre coordinate of the weighted-mean patch - no point state, no sweeps
  const bool nlm_only = P.solver == NLEM_SOLVER_NLM_ONLY;
  const int total_warps = gridDim.x * WARPS;

  // work items: pixels, or (probe launch) probe_n samples at pixel i * plane / probe_n
  const int nidx = probe_n ? probe_n : plane;
  auto pix_of = [&](int i) {
    return probe_n ? static_cast<int>(static_cast<long long>(i) * plane / probe_n) : i;
  };
  int idx = blockIdx.x * WARPS + warp;
  int pix = pix_of(idx);
  auto issue_tile = [&](int p, int b) {
    const int r = out_row0 + p / cols, c = p % cols;
    const float* src = pad + static_cast<int64_t>(r - out_row0) * pad_cols + c;
    (void)b;
    // 87 half-columns of 13 rows (A first / second halves of columns 0..26, B first halves of
    // columns 0..16, B second halves of columns 0..15) in three uniform rounds over the lanes
    // (a branch per copy would serialise the divergent paths)
    auto half = [&](float* dst, const float* sp) {  // 13 rows of one tile column into pair slots
#pragma unroll  // (rolled: 0.55 % slower - the loop control is issued in the serial epilogue)
      for (int e = 0; e < SEGL + KS - 1; ++e, sp += pad_cols) cpa4(dst + 2 * e, sp);
    };
#pragma unroll 1
    for (int rnd = 0; rnd < 3; ++rnd) {
      const int j = rnd * 32 + lane;
      int off, row0, col;
      if (j < TH) { off = PA + j * PCS; row0 = 0; col = j; }
      else if (j < 2 * TH) { off = PA + (j - TH) * PCS + 1; row0 = 7; col = j - TH; }
      else if (j < 2 * TH + BCOLS) { off = PB + (j - 2 * TH) * PCS; row0 = 14; col = j - 2 * TH; }
      else { off = PB + (j - 2 * TH - BCOLS) * PCS + 1; row0 = 14; col = j - 2 * TH - BCOLS + 11; }
      if (j < 2 * TH + BCOLS + BCOLS - 1) half(W + off, src + static_cast<int64_t>(row0) * pad_cols + col);
    }
    cpa_commit();
  };
  // padding pair 13 of every paired column and the second half of B column 16 (tile column 27
  // does not exist) are read by the 16-byte loads but never streamed in: keep them 0
  for (int x = lane; x < TH + BCOLS; x += 32) {
    float* col = W + (x < TH ? PA + x * PCS : PB + (x - TH) * PCS);
    col[26] = 0.0f;
    col[27] = 0.0f;
  }
  if (lane < SEGL + KS - 1) W[PB + 16 * PCS + 2 * lane + 1] = 0.0f;
  // the transpose buffer's rows are summed unconditionally (rows a half does not write hold
  // stale values whose sums every consumer masks): start from defined memory
  for (int e = lane; e < 32 * RED_STR; e += 32) red[e] = 0.0f;
  if (idx < nidx) issue_tile(pix, 0);

#ifdef NLEM_LR_STAMPS
  long long st_t0 = 0, st_t1 = 0, st_t2 = 0, st_t3 = 0, st_wait = 0, st_setup = 0, st_sw = 0, st_epi = 0, st_n = 0;
  long long st_p[4] = {0, 0, 0, 0};
  long long st_s[4] = {0, 0, 0, 0}, st_sq = 0;  // sweep phases: dot, update, patch sum, consensus
  long long st_f[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, st_fq = 0;  // fine stamps
#define LR_FSTAMP(k) { const long long q_ = clock64(); st_f[k] += q_ - st_fq; st_fq = q_; }
#define LR_FSTART() { st_fq = clock64(); }
#else
#define LR_FSTAMP(k)
#define LR_FSTART()
#endif
  while (idx < nidx) {
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(work_counter, 1) + total_warps;
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
#ifdef NLEM_LR_STAMPS
    st_t0 = clock64();
#endif
    cpa_wait();
#ifdef NLEM_LR_STAMPS
    st_t1 = clock64(); st_wait += st_t1 - st_t0;
#endif
    __syncwarp();
    const float* const T = W;

    const int r = out_row0 + pix / cols, c = pix % cols;
    // window of half-width hw = S/2 <= 10 inside the 21 x 21 grid, clipped at the image borders
    // (patch.cpp:72-76); grid points outside it are zero-weight padding points
    const int gr0 = r < hw ? HS - r : wlo;
    const int gr1 = rows - 1 - r < hw ? HS + (rows - 1 - r) : SW - 1 - wlo;
    const int gc0 = c < hw ? HS - c : wlo;
    const int gc1 = cols - 1 - c < hw ? HS + (cols - 1 - c) : SW - 1 - wlo;
    const float inv_n = 1.0f / static_cast<float>((gr1 - gr0 + 1) * (gc1 - gc0 + 1));

#ifdef NLEM_LR_STAMPS
    long long st_q = clock64();
#endif
    // ---- footprint constancy (exact-stop candidate, admm.hpp:77 with tol 0)
    const float a0 = tile_at(T, gr0, gc0);
    bool neq = nlm_only;  // NlmOnly never stops early: no footprint scan
    if (!nlm_only && lane >= gc0 && lane <= gc1 + KS - 1) {
      // column `lane` of the footprint rows [gr0, gr1 + 6]: each column copy b (rows 7b..7b+12)
      // as four independent 16-byte loads (a rolled per-row loop of dependent 4-byte loads
      // cost ~4k cycles per pixel and warp)
      float2 v[14];
      load_pcol(T + PA + lane * PCS, v);  // rows 0..12 (.x) and 7..19 (.y)
#pragma unroll
      for (int q = 0; q < SEGL + KS - 1; ++q) {
        neq |= q >= gr0 && q <= gr1 + KS - 1 && v[q].x != a0;
        neq |= q + 7 >= gr0 && q + 7 <= gr1 + KS - 1 && v[q].y != a0;
      }
      const bool lo = lane < BCOLS;  // rows 14..26 of column `lane` in copy B
      load_pcol(T + PB + (lo ? lane : lane - 11) * PCS, v);
#pragma unroll
      for (int q = 0; q < SEGL + KS - 1; ++q)
        neq |= q + 14 >= gr0 && q + 14 <= gr1 + KS - 1 && (lo ? v[q].x : v[q].y) != a0;
    }
    const bool static_eq = !__any_sync(0xffffffffu, neq);

#ifdef NLEM_LR_STAMPS
    { const long long q_ = clock64(); st_p[0] += q_ - st_q; st_q = q_; }
#endif
    // ---- distances ||a_k - a_self||^2 (patch.cpp:52-61), weights, lambdas; state init
    unsigned realmask = 0;  // bit s*7+i: grid point inside the clipped window (patch.cpp:72-76)
    float2 wgt[SEGL];  // (slot 0, slot 1) pairs
    {
      float2 A2[SEGL];
#pragma unroll
      for (int i = 0; i < SEGL; ++i) A2[i] = make_float2(0.0f, 0.0f);
#pragma unroll 1
      for (int jx = 0; jx < KS; ++jx) {
        float nac[KS];
#pragma unroll
        for (int jy = 0; jy < KS; ++jy) nac[jy] = -tile_at(T, HS + jy, HS + jx);  // a_self
        float2 v[14];
        load_pcol(T + poff + jx * PCS, v);
        p_dist(A2, v, nac);
      }
      float lm[16];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int gx = s ? sgx1 : sgx0, gy0 = s ? sgy01 : sgy00;
        const bool colreal = (s ? sval1 : sval0) && gx >= gc0 && gx <= gc1;
#pragma unroll
        for (int i = 0; i < SEGL; ++i) {
          const float a2 = s ? A2[i].y : A2[i].x;
          const bool real = colreal && gy0 + i >= gr0 && gy0 + i <= gr1;
          const float w = real ? expf(-a2 * P.inv_h2) : 0.0f;  // (ex2.approx: +0.2 %, not taken)
          if (s) wgt[i].y = w; else wgt[i].x = w;
          realmask |= real ? 1u << (s * SEGL + i) : 0u;
          lm[2 * i + s] = irls ? w : inv_mu * w;  // IRLS keeps the weights themselves
        }
      }
      lm[14] = lm[15] = 0.0f;
      if (!nlm_only) {
#pragma unroll
      for (int i = 0; i < SEGL; ++i) {
        // H = ||a~||^2, K = -||a~||^2, ga = 0, ||a~||^2, al = 0 (slot-interleaved)
        const float st[16] = {A2[i].x, A2[i].y, -A2[i].x, -A2[i].y, 0.0f, 0.0f, A2[i].x, A2[i].y,
                              0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        tm_st<16>(t_pt(i), st);
        if constexpr (PC == 32) {  // al_4 .. al_{R-1} = 0
          const float z16[16] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f,
                                 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
          tm_st<16>(t_pt(i) + 16, z16);
        }
      }
      tm_st<16>(t_lam(), lm);
      }
    }
#ifdef NLEM_LR_STAMPS
    { const long long q_ = clock64(); st_p[1] += q_ - st_q; st_q = q_; }
#endif

    // ---- patch-sum pass (sum_k u_k a_k per coordinate) + transpose reduction to the owners.
    // Half A rows (jx - 0) * 7 + jy, half B rows (jx - 4) * 7 + jy, then 5 extra scalars.
    // NEX extra per-lane scalars ride along as rows of their own: all after half B's 21
    // coordinate rows when they fit the 32-row buffer (NEX <= 11), otherwise the first four after
    // half A's 28 rows and the rest after half B's.
    auto patch_sum_reduce = [&]<int NEX>(const float2 (&u2)[SEGL], const float (&extra)[NEX],
                                         float& oA, float& oB, float (&xs)[NEX]) {
      constexpr int EXA = NEX <= 11 ? 0 : 4;  // extras summed with half A
      static_assert(3 * KS + NEX - EXA <= 32, "transpose buffer rows");
      LR_FSTART()
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int jxa = hf ? 4 : 0, jxb = hf ? KS : 4;
        LR_UNROLL(NLEM_LR_UG)
        for (int jx = jxa; jx < jxb; ++jx) {
          float2 g[KS];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy) g[jy] = make_float2(0.0f, 0.0f);
          float2 v[14];
          load_pcol(T + poff + jx * PCS, v);
          p_gsum(g, v, u2);
          float* rrow = red + (jx - jxa) * KS * RED_STR + lane;
#pragma unroll
          for (int jy = 0; jy < KS; ++jy) rrow[jy * RED_STR] = g[jy].x + g[jy].y;
        }
        if (hf) {
#pragma unroll
          for (int q = EXA; q < NEX; ++q) red[(3 * KS + q - EXA) * RED_STR + lane] = extra[q];
        } else {
#pragma unroll
          for (int q = 0; q < EXA; ++q) red[(4 * KS + q) * RED_STR + lane] = extra[q];
        }
        LR_FSTAMP(hf ? 3 : 0)
        __syncwarp();
        LR_FSTAMP(hf ? 4 : 1)
        // every lane sums its row (rows beyond the half's count hold stale, unused values:
        // every consumer is masked by the owner predicates) - no divergent branch
        const float rr = row_sum(red + lane * RED_STR);
        __syncwarp();
        LR_FSTAMP(hf ? 5 : 2)
        if (hf == 0) {
          oA = rr;
#pragma unroll
          for (int q = 0; q < EXA; ++q) xs[q] = __shfl_sync(0xffffffffu, rr, 4 * KS + q);
        } else {
          oB = rr;
#pragma unroll
          for (int q = EXA; q < NEX; ++q) xs[q] = __shfl_sync(0xffffffffu, rr, 3 * KS + q - EXA);
        }
      }
    };

#ifdef NLEM_LR_STAMPS
    { const long long q_ = clock64(); st_p[2] += q_ - st_q; st_q = q_; }
#endif
    // ---- initial patch (nlem.cpp:13-18): weighted mean (ratio form) or the noisy patch.
    // Owner scalars in shared memory: rows 0 z_A, 1 z_B, 2 m_A, 3 m_B, 4.. c~ history ring
    // (slot (head - q) mod (R+1) holds c~_{t-q}), A then B.
    if (nlm_only) {
      // sum_k w_k a_k[centre] / sum_k w_k (nlm.cpp:44): the centre coordinate (3, 3) of point i is
      // row i + 3 of patch column 3; both sums through one butterfly (fixed order)
      float2 v[14];
      load_pcol(T + poff + (KS / 2) * PCS, v);
      float2 cs2 = make_float2(0.0f, 0.0f), ws2 = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < SEGL; ++i) {
        cs2 = __ffma2_rn(wgt[i], v[i + KS / 2], cs2);
        ws2 = __fadd2_rn(ws2, wgt[i]);
      }
      float cs = cs2.x + cs2.y, ws = ws2.x + ws2.y;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        cs += __shfl_xor_sync(0xffffffffu, cs, o);
        ws += __shfl_xor_sync(0xffffffffu, ws, o);
      }
      if (lane == kCenterLane) own[0] = box_clamp(cs / ws, P.range);  // clip_scalar / project_box
    } else {
      const float mA = own0 ? tile_at(T, HS + jy0, HS + jx0) : 0.0f;
      const float mB = own1 ? tile_at(T, HS + jy0, HS + jx1) : 0.0f;
      float zA = mA, zB = mB;
      if (nlm_init) {
        float ex[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int i = 0; i < SEGL; ++i) ex[0] += (s ? wgt[i].y : wgt[i].x);
        float oA, oB, xs[5];
        patch_sum_reduce(wgt, ex, oA, oB, xs);
        zA = own0 ? oA / xs[0] : 0.0f;
        zB = own1 ? oB / xs[0] : 0.0f;
      }
      own[0 * 32] = zA;
      own[1 * 32] = zB;
      own[2 * 32] = mA;
      own[3 * 32] = mB;
#pragma unroll
      for (int q = 1; q <= R; ++q) {
        own[(4 + q) * 32] = 0.0f;
        own[(4 + R + 1 + q) * 32] = 0.0f;
      }
      own[4 * 32] = zA - mA;  // sweep 1: c_1 = z0 (p = z0 - a), centred; head = 0
      own[(4 + R + 1) * 32] = zB - mB;
      if (lane <= R) nrs[lane] = 0.0f;
    }
#ifdef NLEM_LR_STAMPS
    { const long long q_ = clock64(); st_p[3] += q_ - st_q; st_q = q_; }
#endif
    // ring slots: sl[q] holds c~_{t-q} (q < R), sl[R] is the free slot; rotated once per sweep
    int sl[R + 1];
    sl[0] = 0;
#pragma unroll
    for (int q = 1; q <= R; ++q) sl[q] = R + 1 - q;
    // Publish c~_{t+1} and form the Gram row <c~_{t-q}, c~_{t+1}> of the coming sweep.  The row
    // stays in registers (every lane holds the butterfly result) and the owners pass c~_{t+1}, m
    // and the four history vectors they already loaded for the consensus, so only c~ itself goes
    // through shared memory (one __syncwarp): the consensus -> Gram -> dot-product hand-over is a
    // serial chain that no other work of the warp overlaps, so every shared-memory round trip
    // removed from it is time (34.0 vs 32.75 Mpix/s with the prefetched point state).
    // gq = G_0..G_3, ||c~||^2, <m, c~>, ||c~_{t+1-R}||^2.
    float gq[R + 3];
    auto publish_regs = [&](float cA, float cB, float mA, float mB, const float (&hqA)[R],
                            const float (&hqB)[R]) {
      const float nrR = nrs[sl[R]];  // ||c~_{t+1-R}||^2, written R sweeps ago (0 while filling)
      float part[R + 2];
#pragma unroll
      for (int q = 0; q < R; ++q) part[q] = fmaf(hqA[q], cA, hqB[q] * cB);
      part[R] = fmaf(cA, cA, cB * cB);
      part[R + 1] = fmaf(mA, cA, mB * cB);
      if (own0) cb[jx0 * CB_STR + jy0] = cA;
      if (own1) cb[jx1 * CB_STR + jy0] = cB;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < R + 2; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
#pragma unroll
      for (int q = 0; q < R + 2; ++q) gq[q] = part[q];  // same value in every lane
      gq[R + 2] = nrR;
      if (lane == 0) nrs[sl[0]] = part[R];
      __syncwarp();
    };
    tm_wait_st();
    int iters = P.iters;
    int fw = 0x7fffffff;  // first ADMM failure: 2 t (+1 for a non-finite norm)
    bool ovf = false;
    int ifail_iter = -1, ifail_kind = 0;  // IRLS failure record
    if (nlm_only) {
      iters = 0;  // every frame holds the NLM value (nlem.cpp:28-30)
    } else if (irls) {
      // ---- IRLS on the smooth surrogate (proj/include/nlem/irls.hpp:21-68).  Pass p evaluates
      // at x_p: the surrogate S(x_p) = sum w sqrt(||x_p - a||^2 + eps) and beta_k = w_k / sqrt(..),
      // then x_{p+1} = sum beta a / sum beta.  Pass 0 gives `previous`; pass t the iteration-t
      // objective, the stop test (irls.hpp:58) and, if t < T, the next iterate.  Distances are
      // direct differences (no Gram expansion: exact near coincident points, where eps matters).
      float previous = 0.0f;
      int stop_at = -1;
      for (int pass = 0; pass <= P.iters; ++pass) {
        if (own0) cb[jx0 * CB_STR + jy0] = own[0];
        if (own1) cb[jx1 * CB_STR + jy0] = own[32];
        __syncwarp();
        float2 d2[SEGL];
#pragma unroll
        for (int i = 0; i < SEGL; ++i) d2[i] = make_float2(0.0f, 0.0f);
#pragma unroll 1
        for (int jx = 0; jx < KS; ++jx) {
          float nx[KS];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy) nx[jy] = -cb[jx * CB_STR + jy];
          float2 v[14];
          load_pcol(T + poff + jx * PCS, v);
          p_dist(d2, v, nx);
        }
        float2 beta[SEGL];
        float bsum = 0.0f, ssum = 0.0f;
        float wl[16];
        tm_ld16c_wait<PC * SEGL>(tw, wl);
#pragma unroll
        for (int i = 0; i < SEGL; ++i) {
          // one hardware reciprocal square root per point (rsqrt.approx, ~2 ulp)
          const float sx = d2[i].x + P.epsilon, sy = d2[i].y + P.epsilon;
          const float ix = rsq(sx), iy = rsq(sy);
          beta[i] = make_float2(wl[2 * i] * ix, wl[2 * i + 1] * iy);  // irls.hpp:45-46
          bsum += beta[i].x + beta[i].y;
          ssum += fmaf(wl[2 * i], sx * ix, wl[2 * i + 1] * (sy * iy));  // costs.hpp:24-33
        }
        float xA, xB, xs[5];
        {
          const float ex[5] = {bsum, ssum, 0.0f, 0.0f, 0.0f};
          patch_sum_reduce(beta, ex, xA, xB, xs);
        }
        const float den = xs[0], current = xs[1];
        const float xnA = xA / den, xnB = xB / den;
        const bool xbad = __any_sync(0xffffffffu, (own0 && !isfinite(xnA)) || (own1 && !isfinite(xnB)));
        if (!isfinite(current)) {  // non-finite surrogate at x_pass (irls.hpp:39, :52)
          ifail_iter = pass;
          ifail_kind = NLEM_FAIL_IRLS_OBJECTIVE;
          break;
        }
        if (pass >= 1) {
          if (frames != nullptr && lane == kCenterLane)
            frames[static_cast<int64_t>(pass - 1) * plane + pix] = box_clamp(own[0], P.range);
          if (previous - current <= P.irls_tol * fabsf(previous)) {  // irls.hpp:58
            stop_at = pass;
            break;
          }
        }
        previous = current;
        if (pass < P.iters) {
          if (xbad) {  // non-finite x_{pass+1} (irls.hpp:50)
            ifail_iter = pass + 1;
            ifail_kind = NLEM_FAIL_IRLS_ITERATE;
            break;
          }
          if (own0) own[0] = xnA;
          if (own1) own[32] = xnB;
        }
      }
      // the minimiser is x at the stop pass (or x_T), held in own[0/32]
      if (ifail_iter < 0) iters = stop_at > 0 ? stop_at : P.iters;
    } else {
    {
      float zeroR[R];
#pragma unroll
      for (int q = 0; q < R; ++q) zeroR[q] = 0.0f;
      __syncwarp();  // the owners' initial rows (and the cleared norm ring) are visible
      publish_regs(own[4 * 32], own[(4 + R + 1) * 32], own[2 * 32], own[3 * 32], zeroR, zeroR);
    }
#ifdef NLEM_LR_STAMPS
    st_t2 = clock64(); st_setup += st_t2 - st_t1;
#endif
    // small-mu regime (lambda = w / mu against ||p||, e.g. the reference default mu = 1e-3):
    // when the self point's prox scale saturates at sweep 1 (lambda_self = 1/mu >= ||z_0 - a_self||
    // = ||c~_1||), most scales do, no history term decays and the ring would overflow after R
    // sweeps - the pixel goes to the exact kernel right away.  A heuristic: a wrong guess costs
    // time, never accuracy.  Warp-uniform (gq[] holds the same value in every lane).
    if (P.iters > R && !static_eq && inv_mu * inv_mu >= gq[R]) ovf = true;
    for (int t = 1; t <= P.iters && !ovf && !probe_n; ++t) {
      // per slot: (1) dot products D_k = <a_k - m, c~>, (2) scalar update of the 7 points
      // (state in TMEM)
      float2 u[SEGL];  // ga' of (slot 0, slot 1): the FFMA2 pairs of the patch-sum pass
      float vac[R];
#pragma unroll
      for (int q = 0; q < R; ++q) vac[q] = 0.0f;
      float usum = 0.0f;
      bool fnorm = false, sne1 = false;
      float2 Dk2[SEGL];
#ifdef NLEM_LR_STAMPS
      st_sq = clock64();
#endif
      {
#pragma unroll
        for (int i = 0; i < SEGL; ++i) Dk2[i] = make_float2(0.0f, 0.0f);
        LR_UNROLL(NLEM_LR_UD)
        for (int jx = 0; jx < KS; ++jx) {
          float cvx[KS];  // column jx of c~ (two broadcast 16-byte loads)
          {
            const float4 ca = reinterpret_cast<const float4*>(cb + jx * CB_STR)[0];
            const float4 cc = reinterpret_cast<const float4*>(cb + jx * CB_STR)[1];
            cvx[0] = ca.x; cvx[1] = ca.y; cvx[2] = ca.z; cvx[3] = ca.w;
            cvx[4] = cc.x; cvx[5] = cc.y; cvx[6] = cc.z;
          }
          float2 v[14];
          load_pcol(T + poff + jx * PCS, v);
          p_dot(Dk2, v, cvx);
        }
      }
#ifdef NLEM_LR_STAMPS
      { const long long q_ = clock64(); st_s[0] += q_ - st_sq; st_sq = q_; }
#endif
      {
        float lm[16];
        tm_ld16c_wait<PC * SEGL>(tw, lm);
        float G[R];
#pragma unroll
        for (int q = 0; q < R; ++q) G[q] = gq[q];
        const float Gnn = gq[R], Cm = gq[R + 1], nrR = gq[R + 2];
        float2 vac2[R];
#pragma unroll
        for (int q = 0; q < R; ++q) vac2[q] = make_float2(0.0f, 0.0f);
        float2 us2 = make_float2(0.0f, 0.0f);
        const float2 one2 = make_float2(1.0f, 1.0f);
        // non-finite ||p||^2 test (admm.hpp:67-68 via the norm): N * 0 summed over the points is 0
        // unless some N is inf / NaN.  Points with lambda = 0 are included: their N can only turn
        // non-finite through the shared c~ / Gram values, which makes the self point's N (lambda
        // = 1/mu != 0) non-finite in the same sweep, so the flagged sweep is the reference's.
        float2 nchk = make_float2(0.0f, 0.0f);
        float hmax = -1.0f;
        // the state of point pair i + 1 is requested before the arithmetic of pair i
        uint32_t stq[2][PC];
        auto issue_pair = [&](auto ic, uint32_t (&dst)[PC]) {
          constexpr int i = decltype(ic)::value;
          tm::ld16_issue<i * PC>(tw, reinterpret_cast<uint32_t(&)[16]>(dst[0]));
          if constexpr (PC == 32) tm::ld16_issue<i * PC + 16>(tw, reinterpret_cast<uint32_t(&)[16]>(dst[16]));
        };
        auto wait_pair = [&](uint32_t (&dst)[PC]) {
          tm::wait_ld(reinterpret_cast<uint32_t(&)[16]>(dst[0]));
          if constexpr (PC == 32) tm::wait_ld(reinterpret_cast<uint32_t(&)[16]>(dst[16]));
        };
        tm_wait_st();  // the previous sweep's state stores (they had three phases to land)
        issue_pair(std::integral_constant<int, 0>{}, stq[0]);
        static_for<SEGL>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          // point i of both slots as one register pair per field
          float st[PC];
          wait_pair(stq[i & 1]);
#pragma unroll
          for (int q = 0; q < PC; ++q) st[q] = __uint_as_float(stq[i & 1][q]);
          if constexpr (i + 1 < SEGL) issue_pair(std::integral_constant<int, i + 1>{}, stq[(i + 1) & 1]);
          const float2 H = make_float2(st[0], st[1]), K = make_float2(st[2], st[3]);
          const float2 ga = make_float2(st[4], st[5]), a2 = make_float2(st[6], st[7]);
          float2 al[R];
#pragma unroll
          for (int q = 0; q < R; ++q) al[q] = make_float2(st[8 + 2 * q], st[9 + 2 * q]);
          const float2 D_ = __fadd2_rn(Dk2[i], make_float2(-Cm, -Cm));
          float2 X2 = __fmul2_rn(al[R - 1], make_float2(G[R - 1], G[R - 1]));
#pragma unroll
          for (int q = R - 2; q >= 0; --q) X2 = __ffma2_rn(al[q], make_float2(G[q], G[q]), X2);
          const float2 gp1 = __fadd2_rn(ga, one2);
          const float2 t2 = __ffma2_rn(make_float2(-gp1.x, -gp1.y), D_, X2);
          const float2 HG = __fadd2_rn(H, make_float2(Gnn, Gnn));
          const float2 N = __ffma2_rn(make_float2(2.0f, 2.0f), t2, HG);
          float2 sc, Nc;
          {
            const float lx = lm[2 * i], ly = lm[2 * i + 1];
            nchk = __ffma2_rn(N, make_float2(0.0f, 0.0f), nchk);
            Nc = make_float2(fmaxf(N.x, 0.0f), fmaxf(N.y, 0.0f));
            sc.x = lx != 0.0f ? fminf(1.0f, lx * rsq(Nc.x)) : 0.0f;
            sc.y = ly != 0.0f ? fminf(1.0f, ly * rsq(Nc.y)) : 0.0f;
          }
          const float2 B = __fadd2_rn(K, D_);
          const float2 ev = __fmul2_rn(sc, al[R - 1]);
          const float2 evv = __fmul2_rn(__fmul2_rn(ev, ev), make_float2(nrR, nrR));
          // hand-off tests as one running maximum (positive = hand the pixel to the exact
          // kernel), checked once per sweep:
          //  * ring overflow: the dropped term s al_{R-1} c~_{t-R} is above FP32 rounding of p;
          //  * cancellation of the Gram expansion: ||p||^2 far below the terms it is formed from
          //    (N < 2^-8 (H + ||c~||^2)), so FP32 rounding of N would be amplified into s (the
          //    batched kernel's test, kernels_batched_lr.cu).  Padding points (lambda = 0) are
          //    included: a spurious hand-off costs time, never accuracy.
          const float2 vo = __ffma2_rn(Nc, make_float2(-kThr2, -kThr2), evv);
          const float2 vc = __ffma2_rn(HG, make_float2(kCancel, kCancel), make_float2(-N.x, -N.y));
          hmax = max3(hmax, vo.x, vo.y);
          hmax = max3(hmax, vc.x, vc.y);
          float o[PC];
          const float2 oH = __ffma2_rn(sc, __ffma2_rn(sc, Nc, __fmul2_rn(make_float2(-2.0f, -2.0f), B)), a2);
          const float2 oK = __ffma2_rn(sc, B, make_float2(-a2.x, -a2.y));
          const float2 oga = __fmul2_rn(sc, gp1);
          o[0] = oH.x; o[1] = oH.y; o[2] = oK.x; o[3] = oK.y; o[4] = oga.x; o[5] = oga.y;
          o[6] = a2.x; o[7] = a2.y; o[8] = sc.x; o[9] = sc.y;
          vac2[0] = __fadd2_rn(vac2[0], sc);
#pragma unroll
          for (int q = 1; q < R; ++q) {  // al'_q = s al_{q-1}
            const float2 oq = __fmul2_rn(sc, al[q - 1]);
            o[8 + 2 * q] = oq.x;
            o[9 + 2 * q] = oq.y;
            vac2[q] = __fadd2_rn(vac2[q], oq);
          }
          u[i] = oga;
          us2 = __fadd2_rn(us2, oga);
          // two columns per store (wider register tuples fragment the register file: spills)
          static_for<NF>([&](auto qc) {
            constexpr int q = decltype(qc)::value;
            if constexpr (q != 3)  // field 3 (||a~||^2) never changes: not rewritten
              tm_st2c<i * PC + 2 * q>(tw, o[2 * q], o[2 * q + 1]);
          });
        });
#pragma unroll
        for (int q = 0; q < R; ++q) vac[q] = vac2[q].x + vac2[q].y;
        usum = us2.x + us2.y;
        fnorm = !isfinite(nchk.x + nchk.y);
        ovf = hmax > 0.0f;
        if (static_eq) {  // warp-uniform and rare: only an all-equal footprint can stop exactly;
          // the prox scales were just stored as al0 (fields 8 / 9 of each point pair) - reread
          // them from TMEM instead of testing every point in the sweep
          tm_wait_st();
          static_for<SEGL>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            float st[16];
            tm_ld16c_wait<i * PC>(tw, st);
            sne1 |= (((realmask >> i) & 1u) && st[8] != 1.0f) ||
                    (((realmask >> (SEGL + i)) & 1u) && st[9] != 1.0f);
          });
        }
      }
      // a ring overflow / cancellation hands the whole pixel to the exact kernel: stop now
      // (3) g = sum_k ga'_k a_k per coordinate, reduced with usum and the history sums
      float gA, gB, xs[1 + R];
#ifdef NLEM_LR_STAMPS
      { const long long q_ = clock64(); st_s[1] += q_ - st_sq; st_sq = q_; }
#endif
      {
        float ex[1 + R];
        ex[0] = usum;
#pragma unroll
        for (int q = 0; q < R; ++q) ex[1 + q] = vac[q];
        patch_sum_reduce(u, ex, gA, gB, xs);
      }
#ifdef NLEM_LR_STAMPS
      { const long long q_ = clock64(); st_s[2] += q_ - st_sq; st_sq = q_; }
#endif
      // (4) consensus z' = P_C(z - g/n), c = 2 z' - z  (admm.hpp:59-65 in p-form);
      // g_j = sum_q v_q c~_{t-q, j} - (sum_k ga'_k a_kj - U m_j)
      // Every lane loads its (lane-private) owner column - zeros outside the owners - in one
      // batch: z, m and the four history vectors of both halves, which serve the consensus and
      // then the Gram row of the next sweep.  All loads precede all stores (the compiler cannot
      // tell the rows apart and would otherwise serialise the two halves), and the arithmetic is
      // branch-free, so the two halves' dependency chains interleave.
      const int nslot = sl[R];  // the free ring slot receives c~_{t+1}
      float hq[2][R], zr[2], mr[2], zn[2], cn[2];
      zr[0] = own[0];
      zr[1] = own[32];
      mr[0] = own[2 * 32];
      mr[1] = own[3 * 32];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        hq[0][q] = own[(4 + sl[q]) * 32];
        hq[1][q] = own[(4 + R + 1 + sl[q]) * 32];
      }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float g = 0.0f;
#pragma unroll
        for (int q = R - 1; q >= 0; --q) g = fmaf(xs[1 + q], hq[hf][q], g);
        g -= fmaf(-xs[0], mr[hf], hf ? gB : gA);
        const float v = fmaf(-g, inv_n, zr[hf]);
        const float y = v < box_lo ? box_lo : v;  // prox.hpp:45-50 (NaN passes through)
        zn[hf] = box_hi < y ? box_hi : y;
        cn[hf] = (hf ? own1 : own0) ? (2.0f * zn[hf] - zr[hf]) - mr[hf] : 0.0f;
      }
      const bool zbad = (own0 && !isfinite(zn[0])) || (own1 && !isfinite(zn[1]));
      const bool zne = (own0 && zn[0] != a0) || (own1 && zn[1] != a0);
      if (own0) {
        own[0] = zn[0];
        own[(4 + nslot) * 32] = cn[0];
      }
      if (own1) {
        own[32] = zn[1];
        own[(4 + R + 1 + nslot) * 32] = cn[1];
      }
      if (frames != nullptr && lane == kCenterLane)
        frames[static_cast<int64_t>(t - 1) * plane + pix] = zn[0];
      LR_FSTAMP(6)  // xs shuffles + consensus
      // one vote for the rare events; the separate ballots only when one fired
      if (__any_sync(0xffffffffu, zbad | fnorm | ovf)) {
        const unsigned bad_z = __ballot_sync(0xffffffffu, zbad), bad_n = __ballot_sync(0xffffffffu, fnorm);
        const unsigned bad_o = __ballot_sync(0xffffffffu, ovf);
        // a hand-off (ring overflow / cancellation) outranks a failure: the exact kernel redoes
        // the whole pixel and records any failure itself
        if (!bad_o) fw = bad_z ? 2 * t : 2 * t + 1;
        ovf = bad_o != 0u;
        break;
      }
      if (static_eq && !__any_sync(0xffffffffu, sne1 | zne)) {  // residual exactly 0
        iters = t;
        break;
      }
      LR_FSTAMP(7)  // votes
      if (t < P.iters) {
        // rotate the ring: the slot just written becomes c~_{t+1}
#pragma unroll
        for (int q = R; q > 0; --q) sl[q] = sl[q - 1];
        sl[0] = nslot;
        publish_regs(cn[0], cn[1], mr[0], mr[1], hq[0], hq[1]);
      }
      LR_FSTAMP(8)  // publish
#ifdef NLEM_LR_STAMPS
      { const long long q_ = clock64(); st_s[3] += q_ - st_sq; st_sq = q_; }
#endif
    }
    }  // ADMM
    tm_wait_st();
#ifdef NLEM_LR_STAMPS
    st_t3 = clock64(); st_sw += st_t3 - st_t2;
#endif
    const bool any_ovf = __any_sync(0xffffffffu, ovf);
    if (probe_n) {
      if (lane == 0 && any_ovf) atomicAdd(probe_count, 1);
    } else if (any_ovf) {
      // a dropped history term would have been significant: the exact p-form kernel redoes it
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = pix;
    } else if (ifail_iter >= 0) {
      if (lane == 0) record_failure(fail, static_cast<int64_t>(r) * cols + c, ifail_iter, ifail_kind);
    } else if (fw != 0x7fffffff) {
      if (lane == 0) {
        const int tf = fw >> 1;
        const int fail_iter = !(fw & 1) || tf == 1 ? tf : tf - 1;
        record_failure(fail, static_cast<int64_t>(r) * cols + c, fail_iter, NLEM_FAIL_ADMM_ITERATE);
      }
    } else if (lane == kCenterLane) {
      // NLEM-IRLS clips the unconstrained minimiser (nlem.cpp:53-54); ADMM's z is in the box
      const float zc = irls ? box_clamp(own[0], P.range) : own[0];
      out[pix] = zc;
      if (frames)
        for (int t = iters; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pix] = zc;
    }
    __syncwarp();  // every lane is done with the tile before the next one streams in
    if (nxt < nidx) issue_tile(pix_of(nxt), 0);
    idx = nxt;
    pix = pix_of(idx);
#ifdef NLEM_LR_STAMPS
    { const long long e_ = clock64(); st_epi += e_ - st_t3; ++st_n; }
#endif
  }
#ifdef NLEM_LR_STAMPS
  if (blockIdx.x < 2 && lane == 0 && (warp == 0 || warp == 7) && st_n)
    printf("lr stamps blk %d warp %d: pixels %lld tile_wait %lld setup %lld sweeps %lld epilogue %lld (cycles/pixel)\n",
           blockIdx.x, warp, st_n, st_wait / st_n, st_setup / st_n, st_sw / st_n, st_epi / st_n);
  if (blockIdx.x < 2 && lane == 0 && warp == 0 && st_n)
    printf("lr setup: footprint %lld distances+weights+tmem %lld nlm-init(patch sum) %lld owners %lld\n"
           "lr sweeps (all T, cycles/pixel): dot %lld update %lld patch-sum+reduce %lld consensus+publish %lld\n"
           "lr fine: macA %lld syncA %lld rowsumA %lld macB %lld syncB %lld rowsumB %lld consensus %lld votes %lld publish %lld\n",
           st_p[0] / st_n, st_p[1] / st_n, st_p[2] / st_n, st_p[3] / st_n, st_s[0] / st_n, st_s[1] / st_n,
           st_s[2] / st_n, st_s[3] / st_n, st_f[0] / st_n, st_f[1] / st_n, st_f[2] / st_n, st_f[3] / st_n,
           st_f[4] / st_n, st_f[5] / st_n, st_f[6] / st_n, st_f[7] / st_n, st_f[8] / st_n);
#endif
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

#ifndef NLEM_LR_SECONDARY
bool nlem_lr_supported(const NlemLaunch& L) {
  // 32-bit pixel indexing inside the kernel
  const int64_t lim = int64_t(1) << 30;
  return (L.P.solver == NLEM_SOLVER_ADMM || L.P.solver == NLEM_SOLVER_IRLS ||
          L.P.solver == NLEM_SOLVER_NLM_ONLY) && L.P.patch == KS &&
         L.P.search <= SW &&  // smaller (odd) windows run masked inside the 21 x 21 grid
         L.out_rows * L.cols < lim && L.rows < lim && L.pad_cols < lim;
}

bool nlem_lr_probe_wanted(const NlemLaunch& L) {
  return L.P.solver == NLEM_SOLVER_ADMM && L.P.iters > R;
}

cudaError_t launch_nlem_lr(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                           int* probe, cudaStream_t stream) {
  auto kfn = NLEM_LR_NAME;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  const int64_t pixels = L.out_rows * L.cols;
  const int sms = device_caps().sms;
  if (probe != nullptr) {  // probe[0] = predicted hand-offs, probe[1] = the probe's work counter
    const int pn = static_cast<int>(std::min<int64_t>(pixels, kProbe));
    const int64_t pgrid = std::max<int64_t>(1, std::min<int64_t>(sms, (pn + WARPS - 1) / WARPS));
    kfn<<<static_cast<unsigned>(pgrid), WARPS * 32, SMEM_BYTES, stream>>>(
        L.pad, static_cast<int>(L.pad_cols), static_cast<int>(L.rows), static_cast<int>(L.cols),
        static_cast<int>(L.out_row0), static_cast<int>(pixels), L.P, L.out, L.frames, probe + 1,
        ovf_list, ovf_count, L.fail, pn, probe);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(sms, (pixels + WARPS - 1) / WARPS));
  kfn<<<static_cast<unsigned>(grid), WARPS * 32, SMEM_BYTES, stream>>>(
      L.pad, static_cast<int>(L.pad_cols), static_cast<int>(L.rows), static_cast<int>(L.cols),
      static_cast<int>(L.out_row0), static_cast<int>(pixels), L.P, L.out, L.frames, counter,
      ovf_list, ovf_count, L.fail, 0, probe);
  return cudaGetLastError();
}

#else
// The ring-12 build (kernels_nlem_lr_r12.cu): launched after launch_nlem_lr when a probe ran and
// 4 < T <= kLrBigRing; it returns at once unless the probe found the small-mu regime.
cudaError_t launch_nlem_lr_ring12(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                                  int* probe, cudaStream_t stream) {
  static_assert(R == kLrBigRing, "ring length of the secondary build");
  auto kfn = NLEM_LR_NAME;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  const int64_t pixels = L.out_rows * L.cols;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(device_caps().sms, (pixels + WARPS - 1) / WARPS));
  kfn<<<static_cast<unsigned>(grid), WARPS * 32, SMEM_BYTES, stream>>>(
      L.pad, static_cast<int>(L.pad_cols), static_cast<int>(L.rows), static_cast<int>(L.cols),
      static_cast<int>(L.out_row0), static_cast<int>(pixels), L.P, L.out, L.frames, counter,
      ovf_list, ovf_count, L.fail, 0, probe);
  return cudaGetLastError();
}
#endif

}  // namespace nlemk
