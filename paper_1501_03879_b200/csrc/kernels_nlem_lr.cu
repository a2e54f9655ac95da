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
//  * the pixel's 27 x 27 image tile sits in shared memory (row stride 35: the 32 lanes' column
//    segments start on 32 distinct banks), double-buffered: the next pixel's tile streams in
//    with cp.async during the current pixel's sweeps;
//  * lane l owns two vertical segments of 7 grid points (63 segments = 441 points); a column
//    of 13 tile values serves 49 FMAs of the dot products (and of the patch sums);
//  * the per-point state (8 x 32-bit) lives in TENSOR MEMORY: 14 points x 8 columns + 14
//    lambdas per lane = 128 columns per warp, 16 warps = all 512 columns x 128 lanes of the SM,
//    moved with tcgen05.ld/st 32x32b.x8 - registers stay free for the FMA working set;
//  * the 54 per-lane partials (49 coordinates, sum ga, 4 history sums) are reduced with a
//    shared-memory transpose (fixed tree: bitwise deterministic), the 49 consensus coordinates
//    are finished by their owner lanes, which keep z, m and the c~ history in registers; the
//    Gram row <c~_{t-r}, c~_{t+1}> is a 6-value butterfly all-reduce.
#include <algorithm>
#include <cstdlib>

#include "launch.h"

namespace nlemk {

namespace lr {

constexpr int KS = 7, SW = 21, D = KS * KS, HS = SW / 2;
constexpr int TH = SW + KS - 1;  // 27
constexpr int TWS = 35;          // tile row stride (bank-distinct segment starts)
constexpr int TILE = (TH * TWS + 3) / 4 * 4;  // floats per tile buffer (16-byte multiple)
constexpr int WARPS = 16;
constexpr int SEGL = 7;  // points per segment
constexpr int R = 4;     // history ring
constexpr int NF = 8;    // state fields per point in TMEM
constexpr int RED_STR = 36;
constexpr int CB_STR = 8;
// per-warp shared memory (floats)
constexpr int W_TILE0 = 0;
constexpr int W_RED = 2 * TILE;
constexpr int W_CB = W_RED + 32 * RED_STR;
constexpr int W_TOTAL = W_CB + KS * CB_STR;
constexpr size_t SMEM_BYTES = size_t(WARPS) * W_TOTAL * sizeof(float) + 16;
constexpr float kThr2 = 1.0f / 17592186044416.0f;  // (2^-22)^2

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ float rsq(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- TMEM (tcgen05) helpers: 32 lanes x 8 columns of 32-bit per warp access
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
               : "r"(taddr));
  v[0] = __uint_as_float(r0);
  v[1] = __uint_as_float(r1);
  v[2] = __uint_as_float(r2);
  v[3] = __uint_as_float(r3);
  v[4] = __uint_as_float(r4);
  v[5] = __uint_as_float(r5);
  v[6] = __uint_as_float(r6);
  v[7] = __uint_as_float(r7);
}
// Completes all outstanding tcgen05.ld of this thread; the "+f" ties keep every use of the
// loaded registers after the wait (the loads are asynchronous).
__device__ __forceinline__ void tm_wait_ld(float (&v)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]),
                 "+f"(v[7])::"memory");
}
__device__ __forceinline__ void tm_tie(float (&v)[8]) {
  asm volatile(""
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]),
                 "+f"(v[7])::"memory");
}
__device__ __forceinline__ void tm_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float box_clamp(float v, const nlem_box& box) {
  if (!box.bounded) return v;
  const float y = (v < box.lower) ? box.lower : v;
  return (box.upper < y) ? box.upper : y;
}

// Segment geometry: vertical segment (grid column gx, grid rows 7b .. 7b+6).  Slot 0 and slot 1
// of the 32 lanes are chosen so that the 32 segment starts b*7*TWS + gx fall on 32 distinct
// banks in both slots (TWS = 35: 7*35 = 245 = 21 mod 32).
__device__ __forceinline__ void seg_of(int lane, int slot, int& gx, int& gy0, bool& valid) {
  valid = true;
  if (slot == 0) {
    if (lane < 21) { gx = lane; gy0 = 0; }
    else { gx = lane - 21; gy0 = 7; }
  } else {
    if (lane < 10) { gx = 11 + lane; gy0 = 7; }
    else if (lane < 31) { gx = lane - 10; gy0 = 14; }
    else { gx = 0; gy0 = 14; valid = false; }
  }
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
nlem_pixels_lr(const float* __restrict__ pad, int64_t pad_cols, int64_t rows, int64_t cols,
               int64_t out_row0, int64_t out_rows, NlemDevParams P, float* out, float* frames,
               int* work_counter, int* ovf_list, int* ovf_count, FailureSlot* fail) {
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* tm_base_slot = reinterpret_cast<uint32_t*>(smem + WARPS * W_TOTAL);
  float* W = smem + warp * W_TOTAL;
  float* red = W + W_RED;
  float* cb = W + W_CB;

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
                      static_cast<uint32_t>((warp >> 2) * 128);
  auto t_pt = [&](int slot, int i) { return tw + static_cast<uint32_t>((slot * SEGL + i) * NF); };
  auto t_lam = [&](int slot) { return tw + static_cast<uint32_t>(112 + slot * 8); };

  // lane geometry
  int sgx[2], sgy0[2];
  bool svalid[2];
  seg_of(lane, 0, sgx[0], sgy0[0], svalid[0]);
  seg_of(lane, 1, sgx[1], sgy0[1], svalid[1]);
  const bool own1 = lane < D - 32;  // second owned coordinate j = 32 + lane
  const int j0 = lane, j1 = own1 ? 32 + lane : 0;

  const int64_t plane = out_rows * cols;
  const float inv_mu = 1.0f / P.mu;
  const bool nlm_init = P.init_mode == NLEM_INIT_NLM_PATCH;
  const int total_warps = gridDim.x * WARPS;

  int64_t pix = static_cast<int64_t>(blockIdx.x) * WARPS + warp;
  int buf = 0;
  auto issue_tile = [&](int64_t p, int b) {
    const int64_t r = out_row0 + p / cols, c = p % cols;
    const float* src = pad + (r - out_row0) * pad_cols + c;
    float* T = W + W_TILE0 + b * TILE;
    for (int e = lane; e < TH * TH; e += 32) {
      const int tr = e / TH, tc = e - tr * TH;
      cpa4(T + tr * TWS + tc, src + tr * pad_cols + tc);
    }
    cpa_commit();
  };
  if (pix < plane) issue_tile(pix, 0);

  while (pix < plane) {
    int64_t nxt = 0;
    if (lane == 0) nxt = static_cast<int64_t>(atomicAdd(work_counter, 1)) + total_warps;
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    cpa_wait();
    __syncwarp();
    const float* T = W + W_TILE0 + buf * TILE;
    if (nxt < plane) issue_tile(nxt, buf ^ 1);

    const int64_t r = out_row0 + pix / cols, c = pix % cols;
    const int gr0 = r < HS ? static_cast<int>(HS - r) : 0;
    const int gr1 = rows - 1 - r < HS ? static_cast<int>(HS + (rows - 1 - r)) : SW - 1;
    const int gc0 = c < HS ? static_cast<int>(HS - c) : 0;
    const int gc1 = cols - 1 - c < HS ? static_cast<int>(HS + (cols - 1 - c)) : SW - 1;
    const int n = (gr1 - gr0 + 1) * (gc1 - gc0 + 1);
    const float inv_n = 1.0f / static_cast<float>(n);

    // ---- footprint constancy (exact-stop candidate, admm.hpp:77 with tol 0) and a0
    const float ref = T[gr0 * TWS + gc0];
    bool neq = false;
    for (int e = lane; e < TH * TH; e += 32) {
      const int tr = e / TH, tc = e - tr * TH;
      if (tr >= gr0 && tr <= gr1 + KS - 1 && tc >= gc0 && tc <= gc1 + KS - 1)
        neq |= T[tr * TWS + tc] != ref;
    }
    const bool static_eq = !__any_sync(0xffffffffu, neq);

    // ---- self patch m = a_self (grid point (HS, HS)); owners keep m_j
    const float m0 = T[(HS + j0 / KS) * TWS + HS + j0 % KS];
    const float m1 = T[(HS + j1 / KS) * TWS + HS + j1 % KS];

    // ---- distances ||a_k - a_self||^2 (patch.cpp:52-61), weights, lambdas
    float A2[2][SEGL];
    {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int i = 0; i < SEGL; ++i) A2[s][i] = 0.0f;
        const float* col = T + sgy0[s] * TWS + sgx[s];
#pragma unroll 1
        for (int jx = 0; jx < KS; ++jx) {
          float v[SEGL + KS - 1], ac[KS];
#pragma unroll
          for (int e = 0; e < SEGL + KS - 1; ++e) v[e] = col[e * TWS + jx];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy) ac[jy] = T[(HS + jy) * TWS + HS + jx];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy)
#pragma unroll
            for (int i = 0; i < SEGL; ++i) {
              const float df = v[i + jy] - ac[jy];
              A2[s][i] = fmaf(df, df, A2[s][i]);
            }
        }
      }
    }
    float wgt[2][SEGL];
    unsigned realmask = 0;  // bit s*7+i: grid point inside the clipped window (patch.cpp:72-76)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int gx = sgx[s];
      const bool colreal = svalid[s] && gx >= gc0 && gx <= gc1;
#pragma unroll
      for (int i = 0; i < SEGL; ++i) {
        const int gy = sgy0[s] + i;
        const bool real = colreal && gy >= gr0 && gy <= gr1;
        wgt[s][i] = real ? expf(-A2[s][i] * P.inv_h2) : 0.0f;
        realmask |= real ? 1u << (s * SEGL + i) : 0u;
      }
    }
    // state init in TMEM: H = ||a~||^2, K = -||a~||^2, ga = 0, A2, al = 0; lambdas
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int i = 0; i < SEGL; ++i) {
        const float st[8] = {A2[s][i], -A2[s][i], 0.0f, A2[s][i], 0.0f, 0.0f, 0.0f, 0.0f};
        tm_st8(t_pt(s, i), st);
      }
      const float lm[8] = {inv_mu * wgt[s][0], inv_mu * wgt[s][1], inv_mu * wgt[s][2],
                           inv_mu * wgt[s][3], inv_mu * wgt[s][4], inv_mu * wgt[s][5],
                           inv_mu * wgt[s][6], 0.0f};
      tm_st8(t_lam(s), lm);
    }

    // ---- patch-sum pass (sum_k u_k a_k per coordinate) + transpose reduction to the owners.
    // rows: 0..48 coordinates, 49 sum u, 50..53 extra per-lane scalars
    auto patch_sum_reduce = [&](const float (&u)[2][SEGL], const float (&extra)[5], float& own0,
                                float& own1v, float (&xs)[5]) {
      float g[D];
#pragma unroll
      for (int j = 0; j < D; ++j) g[j] = 0.0f;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const float* col = T + sgy0[s] * TWS + sgx[s];
#pragma unroll
        for (int jx = 0; jx < KS; ++jx) {
          float v[SEGL + KS - 1];
#pragma unroll
          for (int e = 0; e < SEGL + KS - 1; ++e) v[e] = col[e * TWS + jx];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy)
#pragma unroll
            for (int i = 0; i < SEGL; ++i) g[jy * KS + jx] = fmaf(u[s][i], v[i + jy], g[jy * KS + jx]);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) red[j * RED_STR + lane] = g[j];
      __syncwarp();
      own0 = row_sum(red + lane * RED_STR);
      __syncwarp();
#pragma unroll
      for (int j = 32; j < D; ++j) red[(j - 32) * RED_STR + lane] = g[j];
#pragma unroll
      for (int q = 0; q < 5; ++q) red[(D - 32 + q) * RED_STR + lane] = extra[q];
      __syncwarp();
      float rb = 0.0f;
      if (lane < D - 32 + 5) rb = row_sum(red + lane * RED_STR);
      __syncwarp();
      own1v = rb;
#pragma unroll
      for (int q = 0; q < 5; ++q) xs[q] = __shfl_sync(0xffffffffu, rb, D - 32 + q);
    };

    // ---- initial patch (nlem.cpp:13-18): weighted mean (ratio form) or the noisy patch
    float z0, z1;
    if (nlm_init) {
      float ex[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < SEGL; ++i) ex[0] += wgt[s][i];
      float o0, o1, xs[5];
      patch_sum_reduce(wgt, ex, o0, o1, xs);
      z0 = o0 / xs[0];
      z1 = o1 / xs[0];
    } else {
      z0 = m0;
      z1 = m1;
    }
    if (!own1) z1 = 0.0f;
    const float mm1 = own1 ? m1 : 0.0f;

    // owner state: c~ history h[0..R] (h[0] = current), squared norms nr[0..R] (uniform)
    float h0[R + 1], h1[R + 1], nr[R + 1];
#pragma unroll
    for (int q = 0; q <= R; ++q) {
      h0[q] = 0.0f;
      h1[q] = 0.0f;
      nr[q] = 0.0f;
    }
    float G[R], Gnn, Cm;
    // publish c~ (owners' h[0]) and the Gram row of the coming sweep
    auto publish = [&]() {
      float part[R + 2];
#pragma unroll
      for (int q = 0; q < R; ++q) part[q] = h0[q + 1] * h0[0] + (own1 ? h1[q + 1] * h1[0] : 0.0f);
      part[R] = h0[0] * h0[0] + (own1 ? h1[0] * h1[0] : 0.0f);
      part[R + 1] = m0 * h0[0] + (own1 ? mm1 * h1[0] : 0.0f);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < R + 2; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
#pragma unroll
      for (int q = 0; q < R; ++q) G[q] = part[q];
      Gnn = part[R];
      Cm = part[R + 1];
#pragma unroll
      for (int q = R; q > 0; --q) nr[q] = nr[q - 1];
      nr[0] = Gnn;
      cb[(j0 / KS) * CB_STR + j0 % KS] = h0[0];
      if (own1) cb[(j1 / KS) * CB_STR + j1 % KS] = h1[0];
      __syncwarp();
    };
    // sweep 1: c_1 = z0 (p = z0 - a), centred
    h0[0] = z0 - m0;
    h1[0] = own1 ? z1 - mm1 : 0.0f;
    publish();
    tm_wait_st();

    const float a0 = ref;
    int iters = P.iters;
    int fw = 0x7fffffff;  // first failure: 2 t (+1 for a non-finite norm)
    bool ovf = false;
    for (int t = 1; t <= P.iters; ++t) {
      // (1) dot products D_k = <a_k - m, c~>
      float Dk[2][SEGL];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < SEGL; ++i) Dk[s][i] = 0.0f;
#pragma unroll
      for (int jx = 0; jx < KS; ++jx) {
        float cvx[KS];  // column jx of c~ (broadcast loads)
#pragma unroll
        for (int jy = 0; jy < KS; ++jy) cvx[jy] = cb[jy * CB_STR + jx];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const float* col = T + sgy0[s] * TWS + sgx[s] + jx;
          float v[SEGL + KS - 1];
#pragma unroll
          for (int e = 0; e < SEGL + KS - 1; ++e) v[e] = col[e * TWS];
#pragma unroll
          for (int jy = 0; jy < KS; ++jy)
#pragma unroll
            for (int i = 0; i < SEGL; ++i) Dk[s][i] = fmaf(v[i + jy], cvx[jy], Dk[s][i]);
        }
      }
      // (2) per-point scalar update (state in TMEM)
      float u[2][SEGL];
      float vac[R] = {0.0f, 0.0f, 0.0f, 0.0f};
      float usum = 0.0f;
      bool fnorm = false, sne1 = false;
      const float Gn = Gnn;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        float lm[8];
        tm_ld8(t_lam(s), lm);
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
        const int i0 = hb * 4, i1 = hb ? SEGL : 4;  // two batches of point loads (registers)
        float st_[4][8];
#pragma unroll
        for (int i = i0; i < i1; ++i) tm_ld8(t_pt(s, i), st_[i - i0]);
        tm_wait_ld(lm);
#pragma unroll
        for (int i = i0; i < i1; ++i) tm_tie(st_[i - i0]);
#pragma unroll
        for (int i = i0; i < i1; ++i) {
          const float (&st_i)[8] = st_[i - i0];
          const float H = st_i[0], K = st_i[1], ga = st_i[2], a2 = st_i[3];
          const float D_ = Dk[s][i] - Cm;
          const float X2 = fmaf(st_i[4], G[0], fmaf(st_i[5], G[1], fmaf(st_i[6], G[2], st_i[7] * G[3])));
          const float N = (H + Gn) + 2.0f * fmaf(-(ga + 1.0f), D_, X2);
          const float lam = lm[i];
          fnorm |= lam != 0.0f && !isfinite(N);
          const float Nc = fmaxf(N, 0.0f);
          const float sc = lam != 0.0f ? fminf(1.0f, lam * rsq(Nc)) : 0.0f;
          sne1 |= ((realmask >> (s * SEGL + i)) & 1u) && sc != 1.0f;
          const float B = K + D_;
          const float ev = sc * st_i[7];
          ovf |= ev * ev * nr[R] > kThr2 * Nc;
          float o[8];
          o[0] = fmaf(sc, fmaf(sc, Nc, -2.0f * B), a2);
          o[1] = fmaf(sc, B, -a2);
          o[2] = sc * (ga + 1.0f);
          o[3] = a2;
          o[4] = sc;
          o[5] = sc * st_i[4];
          o[6] = sc * st_i[5];
          o[7] = sc * st_i[6];
          vac[0] += o[4];
          vac[1] += o[5];
          vac[2] += o[6];
          vac[3] += o[7];
          u[s][i] = o[2];
          usum += o[2];
          tm_st8(t_pt(s, i), o);
        }
        }
      }
      // (3) g = sum_k ga'_k a_k per coordinate, reduced with usum and the history sums
      float ex[5] = {usum, vac[0], vac[1], vac[2], vac[3]};
      float gA0, gA1, xs[5];
      patch_sum_reduce(u, ex, gA0, gA1, xs);
      // (4) consensus z' = P_C(z - g/n), c = 2 z' - z  (admm.hpp:59-65 in p-form)
      const float U = xs[0];
      bool zbad = false, zne = false;
      {
        const float g = fmaf(xs[1], h0[0], fmaf(xs[2], h0[1], fmaf(xs[3], h0[2], xs[4] * h0[3]))) -
                        fmaf(-U, m0, gA0);
        const float zn = box_clamp(fmaf(-g, inv_n, z0), P.range);
        zbad |= !isfinite(zn);
        zne |= zn != a0;
        if (frames != nullptr && j0 == D / 2) frames[static_cast<int64_t>(t - 1) * plane + pix] = zn;
        const float cn = (2.0f * zn - z0) - m0;
#pragma unroll
        for (int q = R; q > 0; --q) h0[q] = h0[q - 1];
        h0[0] = cn;
        z0 = zn;
      }
      if (own1) {
        const float g = fmaf(xs[1], h1[0], fmaf(xs[2], h1[1], fmaf(xs[3], h1[2], xs[4] * h1[3]))) -
                        fmaf(-U, mm1, gA1);
        const float zn = box_clamp(fmaf(-g, inv_n, z1), P.range);
        zbad |= !isfinite(zn);
        zne |= zn != a0;
        const float cn = (2.0f * zn - z1) - mm1;
#pragma unroll
        for (int q = R; q > 0; --q) h1[q] = h1[q - 1];
        h1[0] = cn;
        z1 = zn;
      }
      const unsigned bad_z = __ballot_sync(0xffffffffu, zbad), bad_n = __ballot_sync(0xffffffffu, fnorm);
      if (bad_z | bad_n) {
        fw = bad_z ? 2 * t : 2 * t + 1;
        break;
      }
      if (static_eq && !__any_sync(0xffffffffu, sne1 | zne)) {  // residual exactly 0
        iters = t;
        break;
      }
      if (t < P.iters) {
        tm_wait_st();
        publish();
      }
    }
    tm_wait_st();
    const bool any_ovf = __any_sync(0xffffffffu, ovf);
    if (any_ovf) {
      // a dropped history term would have been significant: the exact p-form kernel redoes it
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = static_cast<int>(pix);
    } else if (fw != 0x7fffffff) {
      if (lane == 0) {
        const int tf = fw >> 1;
        const int fail_iter = !(fw & 1) || tf == 1 ? tf : tf - 1;
        record_failure(fail, r * cols + c, fail_iter, NLEM_FAIL_ADMM_ITERATE);
      }
    } else if (lane == D / 2) {
      out[pix] = z0;
      if (frames)
        for (int t = iters; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pix] = z0;
    }
    pix = nxt;
    buf ^= 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

bool nlem_lr_supported(const NlemLaunch& L) {
  return L.P.solver == NLEM_SOLVER_ADMM && L.P.patch == KS && L.P.search == SW;
}

cudaError_t launch_nlem_lr(const NlemLaunch& L, int* ovf_list, int* ovf_count, int* counter,
                           cudaStream_t stream) {
  auto kfn = nlem_pixels_lr;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(SMEM_BYTES));
  if (e != cudaSuccess) return e;
  const int64_t pixels = L.out_rows * L.cols;
  int64_t grid = device_caps().sms;
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, (pixels + WARPS - 1) / WARPS));
  kfn<<<static_cast<unsigned>(grid), WARPS * 32, SMEM_BYTES, stream>>>(
      L.pad, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out, L.frames, counter,
      ovf_list, ovf_count, L.fail);
  return cudaGetLastError();
}

}  // namespace nlemk
