// Low-rank ("Gram-form") NLEM / EM-ADMM kernel for k = 7, S = 21 (configs 2, 3, 4).
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
// FP32 rounding of p itself.  A pixel whose ring would drop a significant term, or whose
// ||p||^2 expansion cancels, is handed to the exact p-form tile kernel (kernels_nlem_tile.cu)
// through a device-side pixel list.
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
// Mapping (B200): NP horizontally adjacent pixels per warp (NP = 2 for ADMM, the production
// path; NP = 1 for IRLS and the small-mu probe), independent pixel-warps - no CTA barrier on
// the sweep path, so one warp's reduction latency is hidden by the other warps' FMAs.
//  * lane l owns two vertical segments of 7 grid points (63 segments = 441 points) that read
//    the same relative tile offsets, so the pixels' 27 x (27 + NP - 1) union tile sits in shared
//    memory as two PAIRED column-major copies ((slot 0, slot 1) float2 per tile row, see the
//    layout below).  Pixel p's patch column jx is union column jx + p, so one paired-column
//    load (seven 16-byte loads) feeds the FFMA2s of BOTH pixels: at NP = 2, 8 column loads per
//    pass serve 14 pixel-columns instead of 7 per pixel - the shared-memory bytes per MAC, which
//    co-limit the one-pixel kernel with the FMA pipe, drop by 43 % in the two MAC passes;
//  * the per-point state (8 x 32-bit) lives in TENSOR MEMORY: 14 points x 8 columns + 14
//    lambdas per lane = 128 columns per pixel, NP pixels per warp, 16 / NP warps = all 512
//    columns x 128 lanes of the SM - registers stay free for the FMA working set;
//  * the 54 per-lane partials (49 coordinates, sum ga, 4 history sums) of each pixel are reduced
//    with a shared-memory transpose (fixed tree: bitwise deterministic), the 49 consensus
//    coordinates are finished by their owner lanes, which keep z, m and the c~ history in
//    shared memory; the Gram row <c~_{t-r}, c~_{t+1}> is a 6-value butterfly all-reduce.
// The pixels of a warp sweep in lockstep; a pixel that stops (exact stop, failure, hand-off)
// is masked out of the scalar update and the consensus while its partner continues.  Every
// pixel's arithmetic is that of the one-pixel kernel (same operations, same order), so the
// output does not depend on NP or on how the image is split into bands.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "launch.h"

namespace nlemk {

namespace lr {

constexpr int KS = 7, SW = 21, HS = SW / 2;
constexpr int TH = SW + KS - 1;  // 27 tile rows (and columns per pixel)
// Tile layout: two PAIRED column-major copies of the union tile (TH rows x TW = TH + NP - 1
// columns).  A lane's two segments always read the same relative (row, column) offsets, so
// their tile values are stored interleaved as (slot 0, slot 1) float2 pairs and every
// correlation step is one FFMA2 on a pair:
//  * copy A (lanes 0..20: segments (x, grid rows 0..6) and (x, rows 7..13)):
//    A[x][r] = (T[r][x], T[r + 7][x]), r = 0..12, x = 0..TW-1;
//  * copy B (lanes 21..31: segments (x, rows 14..20) and (x + 11, rows 14..20), x = 0..10; lane
//    31's second segment does not exist): B[x][r] = (T[14 + r][x], T[14 + r][x + 11]),
//    x = 0..BCOLS-1 (the second half of the last B column does not exist: kept 0).
// A column is 14 pairs (pair 13 = 0 padding) = seven 16-byte loads; stride PCS = 28 floats (odd
// number of 16-byte quads: 8 consecutive columns hit 8 distinct bank quads) and PB = PA + 12
// mod 32 keeps the LDS.128 phase that straddles the two copies (lanes 16..23) conflict-free.
constexpr int PCS = 28;
constexpr int PA = 0;
constexpr int SEGL = 7;  // points per segment
constexpr int R = 4;     // history ring
constexpr int NF = 8;    // state fields per point in TMEM
constexpr int RED_STR = 36;
constexpr int CB_STR = 8;
constexpr int OWN_ROWS = 4 + 2 * (R + 1);  // z_A, z_B, m_A, m_B, c~ ring A, c~ ring B
constexpr int kProbe = 1024;               // pixels sampled by the small-mu probe launch
constexpr int kCenterLane = 24;            // owner of coordinate D/2 = (3, 3): half A row 3*7+3
constexpr float kThr2 = 1.0f / 17592186044416.0f;  // (2^-22)^2
constexpr float kCancel = 1.0f / 256.0f;  // N below 2^-8 (H + ||c~||^2): the expansion cancels

template <int NP_>
struct Cfg {
  static constexpr int NP = NP_;                       // pixels per warp
  static constexpr int WARPS = 16 / NP;                // pixel-warps per CTA (1 CTA per SM)
  static constexpr int TW = TH + NP - 1;               // union tile width
  static constexpr int BCOLS = 17 + NP - 1;            // copy B columns
  static constexpr int PB = NP == 1 ? 780 : 812;       // copy B base (= 12 mod 32)
  static constexpr int TILE = PB + BCOLS * PCS;        // floats per tile buffer
  static constexpr int NTB = NP == 1 ? 1 : 2;          // tile buffers (double-buffered at NP = 2)
  static constexpr int NHALF = 2 * TW + 2 * BCOLS - 1; // 13-row half-columns streamed per tile
  // per-warp shared memory (floats)
  static constexpr int W_RED = NTB * TILE;
  static constexpr int W_CB = W_RED + NP * 32 * RED_STR;
  static constexpr int W_OWN = W_CB + NP * KS * CB_STR;
  static constexpr int W_NR = W_OWN + NP * OWN_ROWS * 32;  // [NP][R+1 (+pad)] ||c~||^2 ring
  // [NP][8] Gram row of the coming sweep: G[0..R-1], ||c~||^2, <m, c~>, ||c~_{t+1-R}||^2
  static constexpr int W_GR = W_NR + NP * 8;
  static constexpr int W_TOTAL = W_GR + NP * 8;
  static constexpr size_t SMEM_BYTES = size_t(WARPS) * W_TOTAL * sizeof(float) + 16;
  static_assert((PB - PA) % 32 == 12 && PB >= TW * PCS, "copy B placement");
  static_assert(NHALF <= 96, "three rounds of 32 lanes stream a tile");
  static_assert(TILE % 4 == 0 && W_RED % 4 == 0 && W_CB % 4 == 0 && W_TOTAL % 4 == 0,
                "16-byte aligned rows");
};

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
__device__ __forceinline__ void tm_st16(uint32_t taddr, const float* v) {
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
// Base + compile-time column offset (PTX [taddr+imm]): one long-lived base register instead of
// one uniform register per address (those exhausted the uniform register file) or a per-access
// add + R2UR.  Column pairs per store: x8 / x16 register tuples fragment the register file.
template <int OFF>
__device__ __forceinline__ void tm_st2c(uint32_t base, float a, float b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+%1], {%2, %3};" ::"r"(base), "n"(OFF),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b))
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
// the same 16 columns of two pixels' state (two loads, one wait)
template <int OFF>
__device__ __forceinline__ void tm_ld2x16c_wait(uint32_t b0, uint32_t b1, float* v, float* w) {
  uint32_t r[16], q[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32+%34];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33+%34];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
        "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
      : "r"(b0), "r"(b1), "n"(OFF)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = __uint_as_float(r[i]);
    w[i] = __uint_as_float(q[i]);
  }
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

// union-tile element (row r, column x) in the paired copies
template <class C>
__device__ __forceinline__ float tile_at(const float* T, int r, int x) {
  if (r < 13) return T[PA + x * PCS + 2 * r];
  if (r < 20) return T[PA + x * PCS + 2 * (r - 7) + 1];
  return x < C::BCOLS ? T[C::PB + x * PCS + 2 * (r - 14)] : T[C::PB + (x - 11) * PCS + 2 * (r - 14) + 1];
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
// c~ column jx of a pixel (two broadcast 16-byte loads)
__device__ __forceinline__ void load_cvec(const float* cb, int jx, float (&c)[7]) {
  const float4 ca = reinterpret_cast<const float4*>(cb + jx * CB_STR)[0];
  const float4 cc = reinterpret_cast<const float4*>(cb + jx * CB_STR)[1];
  c[0] = ca.x; c[1] = ca.y; c[2] = ca.z; c[3] = ca.w;
  c[4] = cc.x; c[5] = cc.y; c[6] = cc.z;
}

}  // namespace lr

using namespace lr;

// Work items: groups of NP horizontally adjacent pixels of one row (columns NP j .. NP j + NP - 1;
// the last group of a row is short when NP does not divide cols), or (probe launch, NP = 1)
// probe_n sampled pixels.
template <int NP>
__global__ void __launch_bounds__(Cfg<NP>::WARPS * 32, 1)
nlem_pixels_lr(const float* __restrict__ pad, int pad_cols, int rows, int cols, int out_row0,
               int plane, NlemDevParams P, float* out, float* frames, int* work_counter,
               int* ovf_list, int* ovf_count, FailureSlot* fail, int probe_n, int* probe_count) {
  using C = Cfg<NP>;
  constexpr int WARPS = C::WARPS;
  // probe_n > 0 (probe launch): only the setup and the small-mu predictor of probe_n pixels
  // spread evenly over the band, counting predicted hand-offs into *probe_count; no outputs.
  // probe_n == 0 with probe_count (main launch): when more than 90 % of the probe pixels
  // would be handed off (the small-mu regime), every pixel is: *ovf_count = -1 tells the tile
  // kernel to take the whole band, and this launch does no pixel work.  The decision depends on
  // the input only (deterministic).
  if (probe_n == 0 && probe_count != nullptr) {
    const int pt = plane < kProbe ? plane : kProbe;
    if (10 * *static_cast<volatile int*>(probe_count) > 9 * pt) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *ovf_count = -1;
      return;
    }
  }
  extern __shared__ __align__(16) float smem[];
  // warp index through a shuffle: the compiler then knows it is warp-uniform (uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  uint32_t* tm_base_slot = reinterpret_cast<uint32_t*>(smem + WARPS * C::W_TOTAL);
  float* const W = smem + warp * C::W_TOTAL;

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
  // column layout per lane and pixel (128 columns): point pair i (slot 0 and slot 1 point i) =
  // 16 columns, field q of slot s at 2 q + s, so one x16 load yields 8 (slot 0, slot 1) register
  // pairs for the paired (FFMA2 / FMUL2 / FADD2) scalar update; lambdas of the 14 points at
  // 112 + 2 i + s
  const uint32_t tw = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) +
                      static_cast<uint32_t>((warp >> 2) * 128 * NP);

  // lane geometry: segment column offsets in the tile
  int sgx0, sgy00, sgx1, sgy01;
  bool sval0, sval1;
  seg_of(lane, 0, sgx0, sgy00, sval0);
  seg_of(lane, 1, sgx1, sgy01, sval1);
  const int poff = lane < 21 ? PA + lane * PCS : C::PB + (lane - 21) * PCS;  // paired column base
  // coordinate owners: the reduction runs in two halves (patch columns 0-3 and 4-6); row
  // l of half A is coordinate (l % 7, l / 7), row l of half B is (l % 7, 4 + l / 7)
  const bool own0 = lane < 4 * KS, own1 = lane < 3 * KS;
  const int jy0 = lane % KS, jx0 = lane / KS, jx1 = 4 + lane / KS;

  const float inv_mu = 1.0f / P.mu;
  const bool nlm_init = P.init_mode == NLEM_INIT_NLM_PATCH;
  const bool irls = P.solver == NLEM_SOLVER_IRLS;
  const int total_warps = gridDim.x * WARPS;

  // work items: groups of NP adjacent pixels of one row (groups per row = ceil(cols / NP))
  const int gpr = (cols + NP - 1) / NP;
  const int out_rows = plane / cols;
  const int nidx = probe_n ? probe_n : out_rows * gpr;
  auto first_pix = [&](int i) {  // first band pixel of work item i
    if (probe_n) return static_cast<int>(static_cast<long long>(i) * plane / probe_n);
    return (i / gpr) * cols + (i % gpr) * NP;
  };
  int idx = blockIdx.x * WARPS + warp;
  int pix = first_pix(idx);
  int tb = 0;  // tile buffer of the current item
  auto issue_tile = [&](int p0, int buf) {
    const int r = out_row0 + p0 / cols, c = p0 % cols;
    const float* src = pad + static_cast<int64_t>(r - out_row0) * pad_cols + c;
    // the union tile's last column exists only if the group's last pixel does
    const int lastcol = (c + C::TW - 1 < pad_cols) ? C::TW - 1 : pad_cols - 1 - c;
    float* const T = W + buf * C::TILE;
    // NHALF half-columns of 13 rows (A first / second halves of columns 0..TW-1, B first halves
    // of columns 0..BCOLS-1, B second halves of columns 0..BCOLS-2) in three uniform rounds
    // over the lanes (a branch per copy would serialise the divergent paths)
    auto half = [&](float* dst, const float* sp) {  // 13 rows of one tile column into pair slots
#pragma unroll 1
      for (int e = 0; e < SEGL + KS - 1; ++e, sp += pad_cols) cpa4(dst + 2 * e, sp);
    };
#pragma unroll 1
    for (int rnd = 0; rnd < 3; ++rnd) {
      const int j = rnd * 32 + lane;
      int off, row0, col;
      if (j < C::TW) { off = PA + j * PCS; row0 = 0; col = j; }
      else if (j < 2 * C::TW) { off = PA + (j - C::TW) * PCS + 1; row0 = 7; col = j - C::TW; }
      else if (j < 2 * C::TW + C::BCOLS) { off = C::PB + (j - 2 * C::TW) * PCS; row0 = 14; col = j - 2 * C::TW; }
      else { off = C::PB + (j - 2 * C::TW - C::BCOLS) * PCS + 1; row0 = 14; col = j - 2 * C::TW - C::BCOLS + 11; }
      if (j < C::NHALF) half(T + off, src + static_cast<int64_t>(row0) * pad_cols + min(col, lastcol));
    }
    cpa_commit();
  };
  // padding pair 13 of every paired column and the second half of the last B column (tile
  // column TW does not exist) are read by the 16-byte loads but never streamed in: keep them 0
#pragma unroll
  for (int b = 0; b < C::NTB; ++b) {
    float* const T = W + b * C::TILE;
    for (int x = lane; x < C::TW + C::BCOLS; x += 32) {
      float* col = T + (x < C::TW ? PA + x * PCS : C::PB + (x - C::TW) * PCS);
      col[26] = 0.0f;
      col[27] = 0.0f;
    }
    if (lane < SEGL + KS - 1) T[C::PB + (C::BCOLS - 1) * PCS + 2 * lane + 1] = 0.0f;
  }
  if (idx < nidx) issue_tile(pix, 0);

  while (idx < nidx) {
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(work_counter, 1) + total_warps;
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    cpa_wait();
    __syncwarp();
    if constexpr (C::NTB == 2) {  // the next item's tile streams in during this item's sweeps
      if (nxt < nidx) issue_tile(first_pix(nxt), tb ^ 1);
    }
    const float* const T = W + tb * C::TILE;

    const int r = out_row0 + pix / cols, c0 = pix % cols;
    const int gr0 = r < HS ? HS - r : 0;
    const int gr1 = rows - 1 - r < HS ? HS + (rows - 1 - r) : SW - 1;
    // per pixel p of the group: column c0 + p (present if < cols), window columns, n
    bool valid[NP];
    int gc0[NP], gc1[NP];
    float inv_n[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int c = c0 + p;
      valid[p] = c < cols;
      gc0[p] = c < HS ? HS - c : 0;
      gc1[p] = cols - 1 - c < HS ? HS + (cols - 1 - c) : SW - 1;
      inv_n[p] = 1.0f / static_cast<float>((gr1 - gr0 + 1) * (gc1[p] - gc0[p] + 1));
    }

    // ---- footprint constancy (exact-stop candidate, admm.hpp:77 with tol 0): lane x checks
    // union column x; pixel p's footprint is union columns [gc0 + p, gc1 + 6 + p]
    float a0[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) a0[p] = tile_at<C>(T, gr0, gc0[p] + p);
    bool neq[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) neq[p] = false;
    if (lane < C::TW) {
      // column `lane` of the footprint rows [gr0, gr1 + 6]: each column copy as independent
      // 16-byte loads (a rolled per-row loop of dependent 4-byte loads cost ~4k cycles)
      float2 v[14], w[14];
      load_pcol(T + PA + lane * PCS, v);  // rows 0..12 (.x) and 7..19 (.y)
      const bool lo = lane < C::BCOLS;    // rows 14..26 of column `lane` in copy B
      load_pcol(T + C::PB + (lo ? lane : lane - 11) * PCS, w);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const bool colin = lane >= gc0[p] + p && lane <= gc1[p] + KS - 1 + p;
        bool e = false;
#pragma unroll
        for (int q = 0; q < SEGL + KS - 1; ++q) {
          e |= q >= gr0 && q <= gr1 + KS - 1 && v[q].x != a0[p];
          e |= q + 7 >= gr0 && q + 7 <= gr1 + KS - 1 && v[q].y != a0[p];
          e |= q + 14 >= gr0 && q + 14 <= gr1 + KS - 1 && (lo ? w[q].x : w[q].y) != a0[p];
        }
        neq[p] = colin && e;
      }
    }
    bool static_eq[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) static_eq[p] = !__any_sync(0xffffffffu, neq[p]);

    // ---- distances ||a_k - a_self||^2 (patch.cpp:52-61), weights, lambdas; state init.  The
    // self patch column jx of pixel p is union column HS + jx + p, so column x serves pixel p
    // at jx = x - p with the same self values -T[HS + jy][HS + x]
    unsigned realmask[NP];  // bit s*7+i: grid point inside the clipped window (patch.cpp:72-76)
    float2 wgt[NP][SEGL];   // (slot 0, slot 1) pairs
    {
      float2 A2[NP][SEGL];
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int i = 0; i < SEGL; ++i) A2[p][i] = make_float2(0.0f, 0.0f);
#pragma unroll 1
      for (int x = 0; x < KS + NP - 1; ++x) {
        float nac[KS];
#pragma unroll
        for (int jy = 0; jy < KS; ++jy) nac[jy] = -tile_at<C>(T, HS + jy, HS + x);
        float2 v[14];
        load_pcol(T + poff + x * PCS, v);
#pragma unroll
        for (int p = 0; p < NP; ++p)
          if (x - p >= 0 && x - p < KS) p_dist(A2[p], v, nac);
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        float lm[16];
        realmask[p] = 0u;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int gx = s ? sgx1 : sgx0, gy0 = s ? sgy01 : sgy00;
          const bool colreal = valid[p] && (s ? sval1 : sval0) && gx >= gc0[p] && gx <= gc1[p];
#pragma unroll
          for (int i = 0; i < SEGL; ++i) {
            const float a2 = s ? A2[p][i].y : A2[p][i].x;
            const bool real = colreal && gy0 + i >= gr0 && gy0 + i <= gr1;
            const float w = real ? expf(-a2 * P.inv_h2) : 0.0f;
            if (s) wgt[p][i].y = w; else wgt[p][i].x = w;
            realmask[p] |= real ? 1u << (s * SEGL + i) : 0u;
            lm[2 * i + s] = irls ? w : inv_mu * w;  // IRLS keeps the weights themselves
          }
        }
        lm[14] = lm[15] = 0.0f;
#pragma unroll
        for (int i = 0; i < SEGL; ++i) {
          // H = ||a~||^2, K = -||a~||^2, ga = 0, ||a~||^2, al = 0 (slot-interleaved)
          const float st[16] = {A2[p][i].x, A2[p][i].y, -A2[p][i].x, -A2[p][i].y, 0.0f, 0.0f,
                                A2[p][i].x, A2[p][i].y, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
          tm_st16(tw + p * 128 + i * 2 * NF, st);
        }
        tm_st16(tw + p * 128 + 2 * NF * SEGL, lm);
      }
    }

    // ---- patch-sum pass (sum_k u_k a_k per coordinate, every pixel of the group, shared
    // column loads) + transpose reduction to the owners.  Half A rows (jx - 0) * 7 + jy, half B
    // rows (jx - 4) * 7 + jy, then 5 extra scalars per pixel.
    auto patch_sum_reduce = [&](const float2 (&u2)[NP][SEGL], const float (&extra)[NP][5],
                                float (&oA)[NP], float (&oB)[NP], float (&xs)[NP][5]) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int jxa = hf ? 4 : 0, jxb = hf ? KS : 4;
        // rolled: an unrolled column loop made the kernel 30 % larger and 5 % slower
#pragma unroll 1
        for (int x = jxa; x < jxb + NP - 1; ++x) {
          float2 v[14];
          load_pcol(T + poff + x * PCS, v);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const int jx = x - p;
            if (jx < jxa || jx >= jxb) continue;
            float2 g[KS];
#pragma unroll
            for (int jy = 0; jy < KS; ++jy) g[jy] = make_float2(0.0f, 0.0f);
            p_gsum(g, v, u2[p]);
            float* rrow = W + C::W_RED + p * 32 * RED_STR + (jx - jxa) * KS * RED_STR + lane;
#pragma unroll
            for (int jy = 0; jy < KS; ++jy) rrow[jy * RED_STR] = g[jy].x + g[jy].y;
          }
        }
        if (hf) {
#pragma unroll
          for (int p = 0; p < NP; ++p)
#pragma unroll
            for (int q = 0; q < 5; ++q)
              W[C::W_RED + p * 32 * RED_STR + (3 * KS + q) * RED_STR + lane] = extra[p][q];
        }
        __syncwarp();
        float rr[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p)
          rr[p] = lane < (hf ? 3 * KS + 5 : 4 * KS)
                      ? row_sum(W + C::W_RED + p * 32 * RED_STR + lane * RED_STR) : 0.0f;
        __syncwarp();
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (hf == 0) {
            oA[p] = rr[p];
          } else {
            oB[p] = rr[p];
#pragma unroll
            for (int q = 0; q < 5; ++q) xs[p][q] = __shfl_sync(0xffffffffu, rr[p], 3 * KS + q);
          }
        }
      }
    };

    // ---- initial patch (nlem.cpp:13-18): weighted mean (ratio form) or the noisy patch.
    // Owner scalars in shared memory per pixel: rows 0 z_A, 1 z_B, 2 m_A, 3 m_B, 4.. c~
    // history ring (slot (head - q) mod (R+1) holds c~_{t-q}), A then B.
    auto own_of = [&](int p) { return W + C::W_OWN + p * OWN_ROWS * 32 + lane; };
    {
      float zA[NP], zB[NP], mA[NP], mB[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        mA[p] = own0 ? tile_at<C>(T, HS + jy0, HS + jx0 + p) : 0.0f;
        mB[p] = own1 ? tile_at<C>(T, HS + jy0, HS + jx1 + p) : 0.0f;
        zA[p] = mA[p];
        zB[p] = mB[p];
      }
      if (nlm_init) {
        float ex[NP][5];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
#pragma unroll
          for (int q = 0; q < 5; ++q) ex[p][q] = 0.0f;
#pragma unroll
          for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int i = 0; i < SEGL; ++i) ex[p][0] += (s ? wgt[p][i].y : wgt[p][i].x);
        }
        float oA[NP], oB[NP], xs[NP][5];
        patch_sum_reduce(wgt, ex, oA, oB, xs);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          zA[p] = own0 ? oA[p] / xs[p][0] : 0.0f;
          zB[p] = own1 ? oB[p] / xs[p][0] : 0.0f;
        }
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        float* const own = own_of(p);
        own[0 * 32] = zA[p];
        own[1 * 32] = zB[p];
        own[2 * 32] = mA[p];
        own[3 * 32] = mB[p];
#pragma unroll
        for (int q = 1; q <= R; ++q) {
          own[(4 + q) * 32] = 0.0f;
          own[(4 + R + 1 + q) * 32] = 0.0f;
        }
        own[4 * 32] = zA[p] - mA[p];  // sweep 1: c_1 = z0 (p = z0 - a), centred; head = 0
        own[(4 + R + 1) * 32] = zB[p] - mB[p];
        if (lane <= R) W[C::W_NR + p * 8 + lane] = 0.0f;
      }
    }
    int head = 0;
    // publish c~ (owners' ring head) and the Gram row <c~_{t-q}, c~_{t+1}> of the coming sweep
    // for the pixels in `mask` (the butterfly of all NP pixels interleaved)
    auto publish = [&](unsigned mask) {
      float part[NP][R + 2];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float* own = own_of(p);
        const float* hA = own + 4 * 32;
        const float* hB = own + (4 + R + 1) * 32;
        const float cA = hA[head * 32], cB = hB[head * 32];
        const float mA = own[2 * 32], mB = own[3 * 32];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int sl = (head + R - q) % (R + 1);  // c~_{t-q} relative to the new head t+1
          part[p][q] = fmaf(hA[sl * 32], cA, hB[sl * 32] * cB);
        }
        part[p][R] = fmaf(cA, cA, cB * cB);
        part[p][R + 1] = fmaf(mA, cA, mB * cB);
        if ((mask >> p) & 1u) {
          float* const cb = W + C::W_CB + p * KS * CB_STR;
          if (own0) cb[jx0 * CB_STR + jy0] = cA;
          if (own1) cb[jx1 * CB_STR + jy0] = cB;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
          for (int q = 0; q < R + 2; ++q) part[p][q] += __shfl_xor_sync(0xffffffffu, part[p][q], o);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (!((mask >> p) & 1u)) continue;
        float* const gram = W + C::W_GR + p * 8;
#pragma unroll
        for (int q = 0; q < R + 2; ++q) gram[q] = part[p][q];  // same value in every lane
        if (lane == 0) W[C::W_NR + p * 8 + head] = part[p][R];
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int p = 0; p < NP; ++p)  // ||c~_{t+1-R}||^2 (0 while filling)
          if ((mask >> p) & 1u) W[C::W_GR + p * 8 + R + 2] = W[C::W_NR + p * 8 + (head + 1) % (R + 1)];
      }
      __syncwarp();
    };
    tm_wait_st();
    int iters[NP];
    int fw[NP];  // first ADMM failure: 2 t (+1 for a non-finite norm)
    bool ovf[NP];
    int ifail_iter = -1, ifail_kind = 0;  // IRLS failure record (NP = 1)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      iters[p] = P.iters;
      fw[p] = 0x7fffffff;
      ovf[p] = false;
    }
    if constexpr (NP == 1) {
      if (irls) {
        // ---- IRLS on the smooth surrogate (proj/include/nlem/irls.hpp:21-68).  Pass p
        // evaluates at x_p: the surrogate S(x_p) = sum w sqrt(||x_p - a||^2 + eps) and beta_k =
        // w_k / sqrt(..), then x_{p+1} = sum beta a / sum beta.  Pass 0 gives `previous`; pass t
        // the iteration-t objective, the stop test (irls.hpp:58) and, if t < T, the next
        // iterate.  Distances are direct differences (no Gram expansion: exact near coincident
        // points, where eps matters).
        float* const own = own_of(0);
        float* const cb = W + C::W_CB;
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
          float2 beta[1][SEGL];
          float bsum = 0.0f, ssum = 0.0f;
          float wl[16];
          tm_ld16c_wait<2 * NF * SEGL>(tw, wl);
#pragma unroll
          for (int i = 0; i < SEGL; ++i) {
            // one hardware reciprocal square root per point (rsqrt.approx, ~2 ulp)
            const float sx = d2[i].x + P.epsilon, sy = d2[i].y + P.epsilon;
            const float ix = rsq(sx), iy = rsq(sy);
            beta[0][i] = make_float2(wl[2 * i] * ix, wl[2 * i + 1] * iy);  // irls.hpp:45-46
            bsum += beta[0][i].x + beta[0][i].y;
            ssum += fmaf(wl[2 * i], sx * ix, wl[2 * i + 1] * (sy * iy));  // costs.hpp:24-33
          }
          float xA[1], xB[1], xs[1][5];
          {
            const float ex[1][5] = {{bsum, ssum, 0.0f, 0.0f, 0.0f}};
            patch_sum_reduce(beta, ex, xA, xB, xs);
          }
          const float den = xs[0][0], current = xs[0][1];
          const float xnA = xA[0] / den, xnB = xB[0] / den;
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
        if (ifail_iter < 0) iters[0] = stop_at > 0 ? stop_at : P.iters;
      }
    }
    if (!irls) {
      unsigned act = 0;  // pixels still sweeping
#pragma unroll
      for (int p = 0; p < NP; ++p) act |= valid[p] ? 1u << p : 0u;
      publish(act);
      // small-mu regime (lambda = w / mu against ||p||, e.g. the reference default mu = 1e-3):
      // when the self point's prox scale saturates at sweep 1 (lambda_self = 1/mu >= ||z_0 -
      // a_self|| = ||c~_1||), most scales do, no history term decays and the ring would
      // overflow after R sweeps - the pixel goes to the exact kernel right away.  A heuristic:
      // a wrong guess costs time, never accuracy.  Warp-uniform (the Gram row holds the same
      // value in every lane).
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (((act >> p) & 1u) && P.iters > R && !static_eq[p] &&
            inv_mu * inv_mu >= W[C::W_GR + p * 8 + R]) {
          ovf[p] = true;
          act &= ~(1u << p);
        }
      }
      if (probe_n) act = 0;
      for (int t = 1; t <= P.iters && act; ++t) {
        // (1) dot products D_k = <a_k - m, c~> of every pixel (shared column loads)
        float2 Dk2[NP][SEGL];
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
          for (int i = 0; i < SEGL; ++i) Dk2[p][i] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int x = 0; x < KS + NP - 1; ++x) {
          float2 v[14];
          load_pcol(T + poff + x * PCS, v);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const int jx = x - p;
            if (jx < 0 || jx >= KS) continue;
            float cvx[KS];
            load_cvec(W + C::W_CB + p * KS * CB_STR, jx, cvx);
            p_dot(Dk2[p], v, cvx);
          }
        }
        // (2) scalar update of the pixels' 14 points (state in TMEM).  At NP = 2 both pixels'
        // point pair i is loaded by one paired TMEM load and updated together (two independent
        // dependency chains per instruction stream); an inactive pixel's state is dead, so it
        // is updated along with the active one instead of branching.
        float2 u[NP][SEGL];  // ga' of (slot 0, slot 1): the FFMA2 pairs of the patch-sum pass
        float ex[NP][5];     // sum ga', the 4 history sums
        bool fnorm[NP], sne1[NP];
        {
          float lm[NP][16];
          if constexpr (NP == 2) tm_ld2x16c_wait<2 * NF * SEGL>(tw, tw + 128, lm[0], lm[NP - 1]);
          else tm_ld16c_wait<2 * NF * SEGL>(tw, lm[0]);
          float G[NP][R], Gnn[NP], Cm[NP], nrR[NP];
          float2 vac2[NP][R], us2[NP], nchk[NP];
          float hmax[NP];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const float* gram = W + C::W_GR + p * 8;
#pragma unroll
            for (int q = 0; q < R; ++q) G[p][q] = gram[q];
            Gnn[p] = gram[R];
            Cm[p] = gram[R + 1];
            nrR[p] = gram[R + 2];
#pragma unroll
            for (int q = 0; q < R; ++q) vac2[p][q] = make_float2(0.0f, 0.0f);
            us2[p] = nchk[p] = make_float2(0.0f, 0.0f);
            hmax[p] = -1.0f;
          }
          const float2 one2 = make_float2(1.0f, 1.0f);
          static_for<SEGL>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            // point i of both slots as one register pair per field
            float st[NP][16];
            if constexpr (NP == 2) tm_ld2x16c_wait<i * 2 * NF>(tw, tw + 128, st[0], st[NP - 1]);
            else tm_ld16c_wait<i * 2 * NF>(tw, st[0]);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
              const uint32_t tp = tw + p * 128;
              const float2 H = make_float2(st[p][0], st[p][1]), K = make_float2(st[p][2], st[p][3]);
              const float2 ga = make_float2(st[p][4], st[p][5]), a2 = make_float2(st[p][6], st[p][7]);
              const float2 al0 = make_float2(st[p][8], st[p][9]), al1 = make_float2(st[p][10], st[p][11]);
              const float2 al2 = make_float2(st[p][12], st[p][13]), al3 = make_float2(st[p][14], st[p][15]);
              const float2 D_ = __fadd2_rn(Dk2[p][i], make_float2(-Cm[p], -Cm[p]));
              const float2 X2 = __ffma2_rn(al0, make_float2(G[p][0], G[p][0]),
                                __ffma2_rn(al1, make_float2(G[p][1], G[p][1]),
                                __ffma2_rn(al2, make_float2(G[p][2], G[p][2]),
                                           __fmul2_rn(al3, make_float2(G[p][3], G[p][3])))));
              const float2 gp1 = __fadd2_rn(ga, one2);
              const float2 t2 = __ffma2_rn(make_float2(-gp1.x, -gp1.y), D_, X2);
              const float2 HG = __fadd2_rn(H, make_float2(Gnn[p], Gnn[p]));
              const float2 N = __ffma2_rn(make_float2(2.0f, 2.0f), t2, HG);
              // non-finite ||p||^2 test (admm.hpp:67-68 via the norm): N * 0 summed over the
              // points is 0 unless some N is inf / NaN.  Points with lambda = 0 are included:
              // their N can only turn non-finite through the shared c~ / Gram values, which
              // makes the self point's N (lambda = 1/mu != 0) non-finite in the same sweep, so
              // the flagged sweep is the reference's.
              nchk[p] = __ffma2_rn(N, make_float2(0.0f, 0.0f), nchk[p]);
              const float2 Nc = make_float2(fmaxf(N.x, 0.0f), fmaxf(N.y, 0.0f));
              const float lx = lm[p][2 * i], ly = lm[p][2 * i + 1];
              const float2 sc = make_float2(lx != 0.0f ? fminf(1.0f, lx * rsq(Nc.x)) : 0.0f,
                                            ly != 0.0f ? fminf(1.0f, ly * rsq(Nc.y)) : 0.0f);
              const float2 B = __fadd2_rn(K, D_);
              const float2 ev = __fmul2_rn(sc, al3);
              const float2 evv = __fmul2_rn(__fmul2_rn(ev, ev), make_float2(nrR[p], nrR[p]));
              // hand-off tests as one running maximum (positive = hand the pixel to the exact
              // kernel), checked once per sweep:
              //  * ring overflow: the dropped term s al_3 c~_{t-R} is above FP32 rounding of p;
              //  * cancellation of the Gram expansion: ||p||^2 far below the terms it is formed
              //    from (N < 2^-8 (H + ||c~||^2)), so FP32 rounding of N would be amplified into
              //    s (the batched kernel's test, kernels_batched_lr.cu).  Padding points
              //    (lambda = 0) are included: a spurious hand-off costs time, never accuracy.
              const float2 vo = __ffma2_rn(Nc, make_float2(-kThr2, -kThr2), evv);
              const float2 vc = __ffma2_rn(HG, make_float2(kCancel, kCancel), make_float2(-N.x, -N.y));
              hmax[p] = max3(hmax[p], vo.x, vo.y);
              hmax[p] = max3(hmax[p], vc.x, vc.y);
              const float2 oH = __ffma2_rn(sc, __ffma2_rn(sc, Nc, __fmul2_rn(make_float2(-2.0f, -2.0f), B)), a2);
              const float2 oK = __ffma2_rn(sc, B, make_float2(-a2.x, -a2.y));
              const float2 oga = __fmul2_rn(sc, gp1);
              const float2 o1 = __fmul2_rn(sc, al0), o2 = __fmul2_rn(sc, al1), o3 = __fmul2_rn(sc, al2);
              vac2[p][0] = __fadd2_rn(vac2[p][0], sc);
              vac2[p][1] = __fadd2_rn(vac2[p][1], o1);
              vac2[p][2] = __fadd2_rn(vac2[p][2], o2);
              vac2[p][3] = __fadd2_rn(vac2[p][3], o3);
              u[p][i] = oga;
              us2[p] = __fadd2_rn(us2[p], oga);
              tm_st2c<i * 2 * NF + 0>(tp, oH.x, oH.y);
              tm_st2c<i * 2 * NF + 2>(tp, oK.x, oK.y);
              tm_st2c<i * 2 * NF + 4>(tp, oga.x, oga.y);
              tm_st2c<i * 2 * NF + 6>(tp, a2.x, a2.y);
              tm_st2c<i * 2 * NF + 8>(tp, sc.x, sc.y);
              tm_st2c<i * 2 * NF + 10>(tp, o1.x, o1.y);
              tm_st2c<i * 2 * NF + 12>(tp, o2.x, o2.y);
              tm_st2c<i * 2 * NF + 14>(tp, o3.x, o3.y);
            }
          });
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            ex[p][0] = us2[p].x + us2[p].y;
#pragma unroll
            for (int q = 0; q < R; ++q) ex[p][1 + q] = vac2[p][q].x + vac2[p][q].y;
            fnorm[p] = !isfinite(nchk[p].x + nchk[p].y);
            ovf[p] = hmax[p] > 0.0f;
            sne1[p] = false;
            if (static_eq[p] && ((act >> p) & 1u)) {  // warp-uniform and rare: only an all-equal
              // footprint can stop exactly; the prox scales were just stored as al0 (fields 8 / 9
              // of each point pair) - reread them from TMEM instead of testing every point
              tm_wait_st();
              const uint32_t tp = tw + p * 128;
              static_for<SEGL>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                float st[16];
                tm_ld16c_wait<i * 2 * NF>(tp, st);
                sne1[p] |= (((realmask[p] >> i) & 1u) && st[8] != 1.0f) ||
                           (((realmask[p] >> (SEGL + i)) & 1u) && st[9] != 1.0f);
              });
            }
          }
        }
        // (3) g = sum_k ga'_k a_k per coordinate, reduced with usum and the history sums
        float gA[NP], gB[NP], xs[NP][5];
        patch_sum_reduce(u, ex, gA, gB, xs);
        // (4) consensus z' = P_C(z - g/n), c = 2 z' - z  (admm.hpp:59-65 in p-form);
        // g_j = sum_q v_q c~_{t-q, j} - (sum_k ga'_k a_kj - U m_j)
        const int nhead = (head + 1) % (R + 1);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (!((act >> p) & 1u)) continue;
          float* const own = own_of(p);
          bool zbad = false, zne = false;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            if (hf ? own1 : own0) {
              float* h = own + (4 + hf * (R + 1)) * 32;
              const float z = own[hf * 32], m = own[(2 + hf) * 32];
              float g = 0.0f;
#pragma unroll
              for (int q = R - 1; q >= 0; --q) g = fmaf(xs[p][1 + q], h[((head + R + 1 - q) % (R + 1)) * 32], g);
              g -= fmaf(-xs[p][0], m, hf ? gB[p] : gA[p]);
              const float zn = box_clamp(fmaf(-g, inv_n[p], z), P.range);
              zbad |= !isfinite(zn);
              zne |= zn != a0[p];
              if (hf == 0 && frames != nullptr && lane == kCenterLane)
                frames[static_cast<int64_t>(t - 1) * plane + pix + p] = zn;
              own[hf * 32] = zn;
              h[nhead * 32] = (2.0f * zn - z) - m;
            }
          }
          const unsigned bad_z = __ballot_sync(0xffffffffu, zbad), bad_n = __ballot_sync(0xffffffffu, fnorm[p]);
          const unsigned bad_o = __ballot_sync(0xffffffffu, ovf[p]);
          if (bad_z | bad_n | bad_o) {
            // a hand-off (ring overflow / cancellation) outranks a failure: the exact kernel
            // redoes the whole pixel and records any failure itself
            if (!bad_o) fw[p] = bad_z ? 2 * t : 2 * t + 1;
            ovf[p] = bad_o != 0;
            act &= ~(1u << p);
          } else if (static_eq[p] && !__any_sync(0xffffffffu, sne1[p] | zne)) {  // residual exactly 0
            iters[p] = t;
            act &= ~(1u << p);
          }
        }
        if (t < P.iters && act) {
          head = nhead;
          tm_wait_st();
          publish(act);
        }
      }
    }
    tm_wait_st();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (!valid[p]) continue;
      const int pixp = pix + p, cp = c0 + p;
      if (probe_n) {
        if (lane == 0 && ovf[p]) atomicAdd(probe_count, 1);
      } else if (ovf[p]) {
        // a dropped history term would have been significant: the exact p-form kernel redoes it
        if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = pixp;
      } else if (ifail_iter >= 0) {
        if (lane == 0) record_failure(fail, static_cast<int64_t>(r) * cols + cp, ifail_iter, ifail_kind);
      } else if (fw[p] != 0x7fffffff) {
        if (lane == 0) {
          const int tf = fw[p] >> 1;
          const int fail_iter = !(fw[p] & 1) || tf == 1 ? tf : tf - 1;
          record_failure(fail, static_cast<int64_t>(r) * cols + cp, fail_iter, NLEM_FAIL_ADMM_ITERATE);
        }
      } else if (lane == kCenterLane) {
        // NLEM-IRLS clips the unconstrained minimiser (nlem.cpp:53-54); ADMM's z is in the box
        const float zc = irls ? box_clamp(own_of(p)[0], P.range) : own_of(p)[0];
        out[pixp] = zc;
        if (frames)
          for (int t = iters[p]; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pixp] = zc;
      }
    }
    __syncwarp();  // every lane is done with the tile before the next one streams in
    if constexpr (C::NTB == 1) {
      if (nxt < nidx) issue_tile(first_pix(nxt), 0);
    } else {
      tb ^= 1;
    }
    idx = nxt;
    pix = first_pix(idx);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

bool nlem_lr_supported(const NlemLaunch& L) {
  // 32-bit pixel indexing inside the kernel
  const int64_t lim = int64_t(1) << 30;
  return (L.P.solver == NLEM_SOLVER_ADMM || L.P.solver == NLEM_SOLVER_IRLS) && L.P.patch == KS &&
         L.P.search == SW &&
         L.out_rows * L.cols < lim && L.rows < lim && L.pad_cols < lim;
}

bool nlem_lr_probe_wanted(const NlemLaunch& L) {
  return L.P.solver == NLEM_SOLVER_ADMM && L.P.iters > R;
}

namespace {
template <int NP>
cudaError_t launch_lr_np(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                         int probe_n, int* probe, cudaStream_t stream) {
  using C = Cfg<NP>;
  auto kfn = nlem_pixels_lr<NP>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(C::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  const int64_t pixels = L.out_rows * L.cols;
  const int64_t items = probe_n ? probe_n : L.out_rows * ((L.cols + NP - 1) / NP);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(device_caps().sms,
                                                              (items + C::WARPS - 1) / C::WARPS));
  kfn<<<static_cast<unsigned>(grid), C::WARPS * 32, C::SMEM_BYTES, stream>>>(
      L.pad, static_cast<int>(L.pad_cols), static_cast<int>(L.rows), static_cast<int>(L.cols),
      static_cast<int>(L.out_row0), static_cast<int>(pixels), L.P, L.out, L.frames, counter,
      ovf_list, ovf_count, L.fail, probe_n, probe);
  return cudaGetLastError();
}
}  // namespace

#ifndef NLEM_LR_NP
#define NLEM_LR_NP 2  // pixels per warp of the ADMM main launch (A/B build variant np1: 1)
#endif

cudaError_t launch_nlem_lr(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                           int* probe, cudaStream_t stream) {
  const int64_t pixels = L.out_rows * L.cols;
  if (probe != nullptr) {  // probe[0] = predicted hand-offs, probe[1] = the probe's work counter
    const int pn = static_cast<int>(std::min<int64_t>(pixels, kProbe));
    const cudaError_t e = launch_lr_np<1>(L, ovf_list, ovf_count, probe + 1, pn, probe, stream);
    if (e != cudaSuccess) return e;
  }
  // IRLS runs one pixel per warp (its per-pass stop rule is per pixel)
  if (L.P.solver == NLEM_SOLVER_IRLS || NLEM_LR_NP == 1)
    return launch_lr_np<1>(L, ovf_list, ovf_count, counter, 0, probe, stream);
  return launch_lr_np<NLEM_LR_NP>(L, ovf_list, ovf_count, counter, 0, probe, stream);
}

}  // namespace nlemk
