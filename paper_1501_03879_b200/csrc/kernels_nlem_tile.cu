// Tile-reuse NLEM kernel (configs 0, 2, 3): the patch stack is never materialised.
//
// A pixel's S x S window grid of patches (k x k each) is a sliding-window view of one
// (S+k-1)^2 image tile.  Lane (group q, patch row dr) owns KB consecutive grid points
// (gr, gc0..gc0+KB-1) x the k coordinates of patch row dr, so the KB*k elements it touches
// are a_{m,dc} = tile[gr+dr][gc0+m+dc]: only KB+k-1 distinct values.  They are loaded ONCE
// per pixel into registers (as even- and odd-aligned float2 pairs, from two shifted smem
// copies of the tile), next to the p-form state p_{m,dc} (solver_generic.cuh), so a sweep
// reads no point data from shared memory at all.  Per sweep and lane: FADD2/FFMA2 update
// and norm partials over point pairs, a shared-memory transpose of the per-point norm
// partials across the k lanes of the group, one prox scale per lane (rsqrt), a shuffle
// broadcast, g partials, then one CTA barrier and a multi-thread consensus per coordinate.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "launch.h"
#include "solver_generic.cuh"

namespace nlemk {

#ifdef NLEM_PHASE_PROFILE
// Debug-only: clock64 stamps of sweep phases for the first pixels of CTA 0 (warp 0, lane 0
// and the last warp's lane 0), read back by nlem_debug_phase_times.
__device__ long long g_phase[2][64][16];
__device__ long long g_warp[32][64][4];  // per warp lane 0: sweep start, red written, after B1, after B2
#define WSTAMP(slot)                                                                        \
  do {                                                                                     \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && X.dbg_it < 64)                        \
      g_warp[threadIdx.x >> 5][X.dbg_it][slot] = clock64();                                 \
  } while (0)
__device__ long long g_setup[64][8];  // thread 0 of CTA 0: per-pixel setup stamps
#define SSTAMP(slot)                                                                          \
  do {                                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0 && X.dbg_px < 64) g_setup[X.dbg_px][slot] = clock64(); \
  } while (0)
#define PHASE(slot)                                                                            \
  do {                                                                                        \
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == blockDim.x - 32) && X.dbg_it < 64) \
      g_phase[threadIdx.x == 0 ? 0 : 1][X.dbg_it][slot] = clock64();                             \
  } while (0)
#else
#define PHASE(slot) \
  do {              \
  } while (0)
#define WSTAMP(slot) \
  do {               \
  } while (0)
#define SSTAMP(slot) \
  do {               \
  } while (0)
#endif

#ifndef NLEM_XW4_CPT
#define NLEM_XW4_CPT 8
#endif
template <int KS_, int SW_, int KB_, int XW_ = 0>
struct TileCfg {
  static constexpr int KS = KS_;                 // patch side k
  static constexpr int SW = SW_;                 // search window side S
  static constexpr int KB = KB_;                 // grid points per lane (one grid-row segment)
  static constexpr int D = KS * KS;
  static constexpr int G = KS;                   // lanes per group = patch rows
  static constexpr int GPW = 32 / G;             // groups per warp
  static constexpr int NBLK = SW / KB;           // segments per grid row
  static constexpr int NGROUPS = SW * NBLK;
  static constexpr int NGC = NGROUPS;            // groups per CTA (one CTA per pixel)
  static constexpr int WARPS = (NGC + GPW - 1) / GPW;  // point warps
  // consensus mode: 0 = CPT threads per coordinate over all warps between two CTA barriers
  // (k = 5); 4 = split p-form: warp pre-reduction, then CPT threads per coordinate over the
  // warp rows, with the next sweep's state update issued between the consensus loads and
  // their reduction (k = 7)
  static constexpr int XW = XW_;
  // the split form publishes c as KS padded rows of CSTR floats so a lane reads its patch row
  // with 128-bit loads; CSTR/4 odd keeps the 7 row reads of a warp conflict-free
  static constexpr int CSTR = (KS + 3) / 4 * 4 + ((((KS + 3) / 4) % 2) ? 0 : 4);
  static constexpr int CSN = (KS * CSTR + 3) & ~3;
  static constexpr int THREADS = 32 * WARPS;
  // resident CTAs per SM the register budget is capped for: the 2-warp instantiations (11 x 11
  // grids) need many pixels in flight per SM (8 CTAs = 128 registers: k=5/S=11 74 vs 55 Mpix/s
  // at 5 CTAs of 180 registers; 10 and more spill and lose), the 21 x 21 ones are one CTA per SM
  // (k=5 / k=3 on the 21 x 21 grid: 2 / 3 CTAs measured best: 13.9 vs 12.2 and 28.0 vs 25.2 Mpix/s)
  static constexpr int MINB = THREADS <= 64 ? 8 : (THREADS >= 512 ? 1 : (KS == 5 ? 2 : 3));
  static constexpr int KP = KB / 2;              // point pairs per lane
  static constexpr bool ODD = (KB % 2) != 0;     // one unpaired point
  static constexpr int SEG = KB + KS - 1;        // tile values a lane touches
  static constexpr int TH = SW + KS - 1;         // tile side
  static constexpr int TWS = (TH + 4) & ~1;      // tile row stride (even, with slack)
  static constexpr int NE = ((KP - 1 + (KS - 1) / 2) > ((SEG - 1) / 2) ? (KP - 1 + (KS - 1) / 2)
                                                                        : ((SEG - 1) / 2)) + 1;
  static constexpr int NO = KP - 1 + (KS - 2) / 2 + 1;
  // per-lane norm row of the group transpose.  k = 7: 31 = the smallest stride >= KB for which
  // both the row writes (fixed m, 28 lanes) and the column reads (fixed r) are bank-conflict
  // free (a stride of 8 made every write 7-way conflicted); k = 5 has no conflict-free stride
  static constexpr int KBP = (KS == 7 && KB == 7) ? 31 : (KB + 3) & ~3;
  static constexpr int KSP = KS;                 // per-lane coordinate row (unpadded)
  // per-group block of g partials: D floats padded so that CPT consecutive-part blocks land
  // on disjoint bank quads (part * GSTR mod 32 in steps of 4): 52 for D = 49, CPT = 8
  // (split form, D = 49: 56 = the smallest even stride >= D + 2 whose row writes are
  // conflict-free)
  static constexpr int GSTR = (XW_ && D == 49) ? 56
                              : D == 49 ? 52 : ((D + 3) & ~3) + (((((D + 3) & ~3) / 4) % 2) ? 0 : 4);
  // per-warp partial rows (split form): CPT4 = 8 threads read one coordinate from rows part, part+8,
  // ...; a stride of 52 puts the 8 parts on distinct bank quads (56 collided parts p, p+4)
  static constexpr int WSTR = D == 49 ? 52 : GSTR;
  static constexpr int SPL = (KB + G - 1) / G;   // points whose prox scale a lane computes
  static constexpr int CPT = THREADS >= 8 * D ? 8 : THREADS >= 4 * D ? 4 : THREADS >= 2 * D ? 2 : 1;
  static_assert(SW % KB == 0, "segments tile the grid row");
  static_assert(D <= THREADS, "consensus needs one thread per coordinate");
  static_assert(XW == 0 || XW == 4, "consensus modes 0 and 4");
  // XW == 4: threads per coordinate of the consensus over the WARPS warp rows
  static constexpr int CPT4 = NLEM_XW4_CPT;
  static_assert(XW != 4 || (WARPS % CPT4 == 0 && CPT4 * D <= THREADS), "warp rows split evenly");
};

// k = 7 / S = 21 (configs 2, 3, 4; the hand-off target of the low-rank kernel): 63 groups of
// 7 lanes, one CTA of 16 warps per pixel, split p-form.  (Round-1 experiments with a 2-CTA
// cluster per pixel and with dedicated / last-arriving consensus warps measured slower,
// profiles/r1_tile_phase_times.txt; they are not part of the build.)
using TileK7S21 = TileCfg<7, 21, 7, 4>;
using TileK5S11 = TileCfg<5, 11, 11, 0>;   // config 0: 11 groups of 5 lanes, 2 warps
// the remaining odd patch sides up to 7 with windows up to 21 (masked inside the grid when
// smaller): the same template, so no shape with k <= 7 and S <= 21 falls to the generic kernel
using TileK5S21 = TileCfg<5, 21, 7, 0>;    // 63 groups of 5 lanes, 11 warps
using TileK3S11 = TileCfg<3, 11, 11, 0>;   // 11 groups of 3 lanes, 2 warps
using TileK3S21 = TileCfg<3, 21, 7, 0>;    // 63 groups of 3 lanes, 7 warps

template <class C>
struct TileSmem {
  static constexpr int T = C::TH * C::TWS;            // one tile copy
  static constexpr int ROWS = C::NGC * C::G + 40;  // local groups + dummy rows for idle lanes
  static constexpr int NB = (ROWS * C::KBP + 3) & ~3;    // norm transpose (16-byte multiple)
  static constexpr int RED = ((C::NGC + 8) * C::GSTR + C::WARPS * C::WSTR + 3) & ~3;  // g partials per group
                                                   // (+ dummy groups) and per warp (split form)
  static constexpr int TOTAL = 2 * T + NB + RED + C::CSN /*cs*/ + 2 * C::D /*c2*/ + 2 * C::D /*z, a0*/ +
                               C::NGROUPS * C::KBP /*w*/ + 64;
};

__device__ __forceinline__ float2 tf2(float x) { return make_float2(x, x); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 tsub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 tfma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// Per-lane register image of its tile segment t[0..SEG): E[i] = (t[2i], t[2i+1]),
// O[i] = (t[2i+1], t[2i+2]).  a_{m,dc} = t[m+dc].
template <class C>
struct Seg {
  float2 E[C::NE];
  float2 O[C::NO];
  // float2 of the point pair (2q, 2q+1) at coordinate dc
  __device__ __forceinline__ float2 pair(int q, int dc) const {
    return (dc & 1) ? O[q + (dc - 1) / 2] : E[q + dc / 2];
  }
  // the unpaired point m = KB-1 at coordinate dc
  __device__ __forceinline__ float single(int dc) const {
    const int x = C::KB - 1 + dc;
    return (x & 1) ? E[x / 2].y : E[x / 2].x;
  }
};

template <class C>
struct TileCtx {
  float* T0;    // tile
  float* T1;    // tile shifted left by one column
  float* nbuf;  // [NGROUPS][G][KBP]
  float* red;   // [NGC + 8][GSTR] per-group g partials
  float* wred;  // [WARPS][WSTR] per-warp g partials (split form)
  float2* c2;   // [D]
  float* cs;    // [KS][CSTR] c rows (split form)
  float* z;     // [D]
  float* a0;    // [D]
  float* wbuf;  // [NGROUPS][KBP]
  int* flags;   // [4]
  float* scal;  // [32]
  int tid, warp, lane, q, dr, base;
  int grow0;    // first transpose/partial row of the lane's group (dummy rows if idle)
  bool active;  // lane belongs to a real group
  bool slot;    // lane belongs to a group slot (lanes past GPW * G of a warp are idle)
  int gr, gc0;  // grid row and first grid column of the lane's segment

  int nloc;        // real groups (the pixel's 63 segments)
  int dbg_it = 0;  // debug phase-profile sweep counter
  int dbg_px = 0;  // debug setup-profile pixel counter
  __device__ void carve(float* smem) {
    T0 = smem;
    T1 = T0 + TileSmem<C>::T;
    nbuf = T1 + TileSmem<C>::T;
    red = nbuf + TileSmem<C>::NB;
    wred = red + (C::NGC + 8) * C::GSTR;
    cs = red + TileSmem<C>::RED;
    c2 = reinterpret_cast<float2*>(cs + C::CSN);
    z = reinterpret_cast<float*>(c2 + C::D);
    a0 = z + C::D;
    wbuf = a0 + C::D;
    flags = reinterpret_cast<int*>(wbuf + C::NGROUPS * C::KBP);
    scal = reinterpret_cast<float*>(flags + 8);
    tid = threadIdx.x;
    warp = tid >> 5;
    lane = tid & 31;
    const int ql = lane / C::G;
    dr = lane - ql * C::G;
    base = ql * C::G;
    const int lq = warp * C::GPW + ql;  // group
    q = lq;
    nloc = C::NGROUPS;
    active = ql < C::GPW && lq < nloc;
    slot = ql < C::GPW;
    // lanes of a group slot without a real group keep their slot's rows (all-zero partials, so
    // per-warp sums over GPW rows stay exact); lanes outside any slot get private dummy rows
    grow0 = ql < C::GPW ? lq * C::G : C::NGC * C::G + base;
    const int qq = active ? q : 0;
    gr = qq / C::NBLK;
    gc0 = (qq % C::NBLK) * C::KB;
  }
};

// Transpose-reduce per-point partials across the G lanes of a group through shared memory:
// v[m] = this lane's partial for point m (m < KB); returns, for the SPL points m = dr + i*G
// this lane owns, the group totals.  Fixed summation order (lanes 0..G-1).
template <class C>
__device__ __forceinline__ float tree_sum_col(const float* col, int stride) {
  float v[C::G];
#pragma unroll
  for (int r = 0; r < C::G; ++r) v[r] = col[r * stride];
#pragma unroll
  for (int w = 1; w < C::G; w <<= 1)
#pragma unroll
    for (int r = 0; r + w < C::G; r += 2 * w) v[r] += v[r + w];
  return v[0];
}

template <class C>
__device__ __forceinline__ void group_point_totals(TileCtx<C>& X, const float (&v)[C::KB],
                                                   float (&tot)[C::SPL]) {
  // lanes outside a group slot skip the exchange: their dummy rows shared banks with real rows
  float* row = X.nbuf + (X.grow0 + X.dr) * C::KBP;
  if (X.slot) {
#pragma unroll
    for (int m = 0; m < C::KB; ++m) row[m] = v[m];
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < C::SPL; ++i) {
    const int m = X.dr + i * C::G;
    tot[i] = X.slot && (C::SPL == 1 || m < C::KB)
                 ? tree_sum_col<C>(X.nbuf + X.grow0 * C::KBP + (m < C::KB ? m : 0), C::KBP)
                 : 0.0f;
  }
  __syncwarp();
}

// Broadcast per-point values (owned by lane m % G, slot m / G) to every lane of the group.
template <class C>
__device__ __forceinline__ void group_broadcast(const TileCtx<C>& X, const float (&own)[C::SPL],
                                                float (&all)[C::KB]) {
#pragma unroll
  for (int m = 0; m < C::KB; ++m) {
    float v = own[0];
#pragma unroll
    for (int i = 1; i < C::SPL; ++i)
      if (m / C::G == i) v = own[i];
    all[m] = __shfl_sync(0xffffffffu, v, X.base + m % C::G);
  }
}

// Sum the per-lane coordinate partials v[dc] (coordinate j = dr*KS + dc) over all groups:
// lanes write red[lq][dr][dc]; after a barrier CPT threads per coordinate sum this CTA's
// groups in a fixed order.  `finish(j, total)` runs on one thread per coordinate.  Ends with a
// CTA barrier.
template <class C, class Finish>
__device__ __forceinline__ void reduce_coordinates(TileCtx<C>& X, const float (&v)[C::KS],
                                                   Finish finish) {
  {
    float* row = X.red + (X.grow0 / C::G) * C::GSTR + X.dr * C::KS;  // idle lanes: dummy groups
#pragma unroll
    for (int dc = 0; dc < C::KS; ++dc) row[dc] = v[dc];
  }
  WSTAMP(1);
  __syncthreads();
  WSTAMP(2);
  PHASE(6);
  const int j = X.tid / C::CPT, part = X.tid % C::CPT;
  float s = 0.0f;
  if (j < C::D) {
    const float* col = X.red + part * C::GSTR + j;
    // all loads first (independent), then a fixed-order pairwise tree
    constexpr int NPER = (C::NGC + C::CPT - 1) / C::CPT;
    float v[NPER];
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      v[i] = (part + i * C::CPT < X.nloc) ? col[i * C::CPT * C::GSTR] : 0.0f;
#pragma unroll
    for (int w = 1; w < NPER; w <<= 1)
#pragma unroll
      for (int i = 0; i + w < NPER; i += 2 * w) v[i] += v[i + w];
    s = v[0];
  }
  PHASE(7);
#pragma unroll
  for (int o = 1; o < C::CPT; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  PHASE(8);
  PHASE(11);
  if (j < C::D && part == 0) finish(j, s);
  PHASE(9);
  __syncthreads();
  WSTAMP(3);
  PHASE(10);
}

// IRLS consensus: lanes write their num partials v[dc] (coordinate j = dr*KS + dc)
// and one lane per group writes the group's sum beta and sum w*root into columns D and D+1 of
// the group row (GSTR >= D + 2).  CPT threads per coordinate sum the 3 columns over groups in
// a fixed order; finish(j, num, den, sur) runs on one thread per coordinate.
template <class C, class Finish>
__device__ __forceinline__ void irls_reduce(TileCtx<C>& X, const float (&v)[C::KS], float gden,
                                            float gsur, Finish finish) {
  static_assert(C::GSTR >= C::D + 2, "room for the den / surrogate columns");
  if (X.slot) {  // (lanes outside a group slot: dummy rows, never read)
    float* row = X.red + (X.grow0 / C::G) * C::GSTR;
#pragma unroll
    for (int dc = 0; dc < C::KS; ++dc) row[X.dr * C::KS + dc] = v[dc];
    if (X.dr == 0) {
      row[C::D] = gden;
      row[C::D + 1] = gsur;
    }
  }
  __syncthreads();
  const int j = X.tid / C::CPT, part = X.tid % C::CPT;
  float sn = 0.0f, sd = 0.0f, ss = 0.0f;
  if (j < C::D) {
    constexpr int NPER = (C::NGC + C::CPT - 1) / C::CPT;
    float a[NPER], b[NPER], c[NPER];
#pragma unroll
    for (int i = 0; i < NPER; ++i) {
      const bool ok = part + i * C::CPT < X.nloc;
      const float* g = X.red + (part + i * C::CPT) * C::GSTR;
      a[i] = ok ? g[j] : 0.0f;
      b[i] = ok ? g[C::D] : 0.0f;
      c[i] = ok ? g[C::D + 1] : 0.0f;
    }
#pragma unroll
    for (int w = 1; w < NPER; w <<= 1)
#pragma unroll
      for (int i = 0; i + w < NPER; i += 2 * w) {
        a[i] += a[i + w];
        b[i] += b[i + w];
        c[i] += c[i + w];
      }
    sn = a[0];
    sd = b[0];
    ss = c[0];
  }
#pragma unroll
  for (int o = 1; o < C::CPT; o <<= 1) {
    sn += __shfl_xor_sync(0xffffffffu, sn, o);
    sd += __shfl_xor_sync(0xffffffffu, sd, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (j < C::D && part == 0) finish(j, sn, sd, ss);
  __syncthreads();
}

// CTA-wide sum of one scalar per lane (fixed order: warp tree, then warps).
template <class C>
__device__ __forceinline__ float block_sum_scalar(TileCtx<C>& X, float v) {
  v = warp_sum(v);
  if (X.lane == 0) X.scal[X.warp] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int w = 0; w < C::WARPS; ++w) t += X.scal[w];
  __syncthreads();
  return t;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
nlem_pixels_tile(const float* __restrict__ pad, int64_t pad_cols, int64_t rows, int64_t cols,
                 int64_t out_row0, int64_t out_rows, NlemDevParams P, float* out, float* frames,
                 int* work_counter, int chunk, FailureSlot* fail, const int* list,
                 const int* list_count) {
  extern __shared__ __align__(16) float smem[];
  TileCtx<C> X;
  X.carve(smem);
  __shared__ long long s_next_chunk[2];  // this CTA's next chunk (double-buffered)
  int chunk_parity = 0;
  constexpr int hs = C::SW / 2;
  const int hw = P.search / 2, wlo = hs - hw;  // masked window (S <= SW)
  constexpr int center = C::D / 2;
  const int64_t plane = out_rows * cols;
  // list mode: only the listed band pixels (the low-rank kernel's hand-offs), in list order
  // (a count of -1: the low-rank kernel handed off the whole band - the small-mu probe)
  const int lcount = list ? *list_count : 0;
  if (lcount < 0) {  // whole band: chunks of up to 8 pixels as in a direct launch
    list = nullptr;
    const int64_t c8 = plane / (static_cast<int64_t>(gridDim.x) * 4);
    chunk = static_cast<int>(c8 < 1 ? 1 : c8 > 8 ? 8 : c8);
  }
  const int64_t npix = list ? static_cast<int64_t>(lcount) : plane;
  const int64_t nchunks = (npix + chunk - 1) / chunk;
  auto pixel_at = [&](int64_t q) -> int64_t { return list ? static_cast<int64_t>(list[q]) : q; };
  const float inv_mu = 1.0f / P.mu;
  // lane-constant tile addressing of the segment (row gr+dr, columns gc0..gc0+SEG)
  const int trow = X.gr + X.dr;
  const bool even = (X.gc0 & 1) == 0;
  const int offE = trow * C::TWS + (even ? X.gc0 : X.gc0 - 1);
  const int offO = trow * C::TWS + (even ? X.gc0 : X.gc0 + 1);
  const bool useT1E = !even, useT1O = even;
  // zero the tile slack columns once
  for (int e = X.tid; e < 2 * TileSmem<C>::T; e += C::THREADS) X.T0[e] = 0.0f;
  __syncthreads();

  // pixel chunks: a CTA takes chunk blockIdx.x, then grabs the next one from a global counter
  // at the start of each chunk (dynamic, so a slow SM does not stretch the launch)
  const int64_t cid = blockIdx.x, ncl = gridDim.x;
  int64_t prefetched = -1;  // pixel whose tile is already in flight to smem
  for (int64_t ch = cid; ch < nchunks;) {
    const int64_t q_end = (ch + 1) * chunk < npix ? (ch + 1) * chunk : npix;
    // read after this chunk's first barrier; rewritten only after the chunk's last one
    // (double-buffered: a slow reader of the previous slot can still be before its barrier)
    if (X.tid == 0) s_next_chunk[chunk_parity] = ncl + atomicAdd(work_counter, 1);
    const auto next_chunk = [&]() -> int64_t { return s_next_chunk[chunk_parity]; };
    for (int64_t q = ch * chunk; q < q_end; ++q) {
      const int64_t pix = pixel_at(q);
      const int64_t r = out_row0 + pix / cols, c = pix % cols;
      // window of half-width hw = S/2 <= hs inside the kernel's SW x SW grid, clipped at the
      // image borders (patch.cpp:72-76); grid points outside it are zero-weight padding
      const int gr0 = r < hw ? static_cast<int>(hs - r) : wlo;
      const int gr1 = rows - 1 - r < hw ? static_cast<int>(hs + (rows - 1 - r)) : C::SW - 1 - wlo;
      const int gc0w = c < hw ? static_cast<int>(hs - c) : wlo;
      const int gc1w = cols - 1 - c < hw ? static_cast<int>(hs + (cols - 1 - c)) : C::SW - 1 - wlo;
      const int n = (gr1 - gr0 + 1) * (gc1w - gc0w + 1);
      const float inv_n = 1.0f / static_cast<float>(n);
      // ---- tile (and its one-column-shifted copy) from the padded band; after the first
      // pixel it was prefetched with cp.async during the previous pixel's sweeps
      SSTAMP(0);
      if (prefetched == pix) {
        cp_async_wait_all();
      } else {
        const float* src = pad + (r - out_row0) * pad_cols + c;
        for (int e = X.tid; e < C::TH * C::TH; e += C::THREADS) {
          const int tr = e / C::TH, tc = e - tr * C::TH;
          const float v = __ldg(src + tr * pad_cols + tc);
          X.T0[tr * C::TWS + tc] = v;
          if (tc > 0) X.T1[tr * C::TWS + tc - 1] = v;
        }
      }
      __syncthreads();
      // footprint-constancy (all real patches equal <=> exact-stop candidate) and a0
      const float ref = X.T0[gr0 * C::TWS + gc0w];
      int neq = 0;
      for (int e = X.tid; e < C::TH * C::TH; e += C::THREADS) {
        const int tr = e / C::TH, tc = e - tr * C::TH;
        if (tr >= gr0 && tr <= gr1 + C::KS - 1 && tc >= gc0w && tc <= gc1w + C::KS - 1)
          neq |= X.T0[tr * C::TWS + tc] != ref;
      }
      if (X.tid < C::D) X.a0[X.tid] = ref;
      if (X.tid == 0) {
        X.flags[0] = 0;
        X.flags[1] = 0;
        X.flags[2] = 0;
        X.flags[3] = 0;
        X.flags[4] = 0x7fffffff;  // XW == 4: first failing sweep (2 t + [no non-finite z])
      }
      // ---- segment registers
      Seg<C> S;
      {
        const float2* pE = reinterpret_cast<const float2*>((useT1E ? X.T1 : X.T0) + offE);
        const float2* pO = reinterpret_cast<const float2*>((useT1O ? X.T1 : X.T0) + offO);
#pragma unroll
        for (int i = 0; i < C::NE; ++i) S.E[i] = pE[i];
#pragma unroll
        for (int i = 0; i < C::NO; ++i) S.O[i] = pO[i];
      }
      SSTAMP(1);
      const bool static_eq = !__syncthreads_or(neq);
      SSTAMP(2);
      // is grid point m of my segment a real neighbour (inside the clipped window)?
      const bool row_real = X.active && X.gr >= gr0 && X.gr <= gr1;
      auto is_real = [&](int m) {
        const int gc = X.gc0 + m;
        return row_real && m < C::KB && gc >= gc0w && gc <= gc1w;
      };
      // ---- similarity weights w_m = exp(-||P_m - P_self||^2 / h^2)  (patch.cpp:52-61)
      float wown[C::SPL];
      {
        float sv[C::KS];
#pragma unroll
        for (int dc = 0; dc < C::KS; ++dc) sv[dc] = X.T0[(hs + X.dr) * C::TWS + hs + dc];
        float d2[C::KB];
#pragma unroll
        for (int qq = 0; qq < C::KP; ++qq) {
          float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) {
            const float2 e = tsub2(S.pair(qq, dc), tf2(sv[dc]));
            acc = tfma2(e, e, acc);
          }
          d2[2 * qq] = acc.x;
          d2[2 * qq + 1] = acc.y;
        }
        if (C::ODD) {
          float acc = 0.0f;
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) {
            const float e = S.single(dc) - sv[dc];
            acc = fmaf(e, e, acc);
          }
          d2[C::KB - 1] = acc;
        }
        float tot[C::SPL];
        group_point_totals<C>(X, d2, tot);
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) {
          const int m = X.dr + i * C::G;
          wown[i] = is_real(m) ? expf(-tot[i] * P.inv_h2) : 0.0f;
        }
      }
      float wall[C::KB];
      group_broadcast<C>(X, wown, wall);
      SSTAMP(3);
      // ---- initial patch (nlem.cpp:13-18)
      const bool nlm_init = P.solver == NLEM_SOLVER_NLM_ONLY || P.init_mode == NLEM_INIT_NLM_PATCH;
      bool init_done = false;
      {
        if (nlm_init) {
          // sum_k w_k a_k / sum_k w_k with the weight sum riding along as an extra consensus
          // column (one reduction, no separate W pass); algebraically the reference's
          // points * (w / sum w) (types.hpp:73), exact for constant integer images
          float v[C::KS];
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) {
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int k = 0; k < C::KP; ++k)
              acc = tfma2(make_float2(wall[2 * k], wall[2 * k + 1]), S.pair(k, dc), acc);
            float t = acc.x + acc.y;
            if (C::ODD) t = fmaf(wall[C::KB - 1], S.single(dc), t);
            v[dc] = X.active ? t : 0.0f;
          }
          float gw = 0.0f;
#pragma unroll
          for (int m = 0; m < C::KB; ++m) gw += wall[m];
          irls_reduce<C>(X, v, X.active ? gw : 0.0f, 0.0f,
                         [&](int j, float num, float den, float) { X.z[j] = num / den; });
          init_done = true;
        }
      }
      if (init_done) {
      } else if (nlm_init) {
        // W = sum of weights (each point counted once by its owner lane)
        float wsum = 0.0f;
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) wsum += wown[i];
        const float W = block_sum_scalar<C>(X, X.active ? wsum : 0.0f);
        const bool ratio = P.nlm_ratio != 0;
        float coef[C::KB];
#pragma unroll
        for (int m = 0; m < C::KB; ++m) coef[m] = ratio ? wall[m] : wall[m] / W;  // points*(w/sum w)
        float v[C::KS];
#pragma unroll
        for (int dc = 0; dc < C::KS; ++dc) {
          float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int qq = 0; qq < C::KP; ++qq)
            acc = tfma2(make_float2(coef[2 * qq], coef[2 * qq + 1]), S.pair(qq, dc), acc);
          float t = acc.x + acc.y;
          if (C::ODD) t = fmaf(coef[C::KB - 1], S.single(dc), t);
          v[dc] = X.active ? t : 0.0f;
        }
        reduce_coordinates<C>(X, v, [&](int j, float tsum) { X.z[j] = ratio ? tsum / W : tsum; });
      } else {
        if (X.tid < C::D) {
          const int jr = X.tid / C::KS, jc = X.tid - jr * C::KS;
          X.z[X.tid] = X.T0[(hs + jr) * C::TWS + hs + jc];
        }
        __syncthreads();
      }

      SSTAMP(4);
      // prefetch the next pixel's tile while this pixel's sweeps run (the tile is only read
      // during the setup above, which ended with a barrier)
      {
        int64_t nq = q + 1;
        if (nq >= q_end) nq = next_chunk() < nchunks ? next_chunk() * chunk : -1;
        const int64_t nxt = nq >= 0 ? pixel_at(nq) : -1;
        if (nxt >= 0) {
          const int64_t nr_ = out_row0 + nxt / cols, nc_ = nxt % cols;
          const float* nsrc = pad + (nr_ - out_row0) * pad_cols + nc_;
          for (int e = X.tid; e < C::TH * C::TH; e += C::THREADS) {
            const int tr = e / C::TH, tc = e - tr * C::TH;
            cp_async4(&X.T0[tr * C::TWS + tc], nsrc + tr * pad_cols + tc);
            if (tc > 0) cp_async4(&X.T1[tr * C::TWS + tc - 1], nsrc + tr * pad_cols + tc);
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
          prefetched = nxt;
        }
      }
      SSTAMP(5);
      int iters = P.iters, fail_iter = -1, fail_kind = 0;
      {
        if (P.solver == NLEM_SOLVER_IRLS) {
          // ---- IRLS on the smooth surrogate (proj/include/nlem/irls.hpp:21-68): pass p
          // evaluates at x_p: surrogate S(x_p) and beta_k = w_k / sqrt(||x_p - a_k||^2 + eps),
          // then x_{p+1} = sum beta a / sum beta.  Pass 0 gives `previous`; pass t gives the
          // iteration-t objective, the stop test and (if t < T) the next iterate.
          float wown0 = wown[0];
          float previous = 0.0f;
          int stop_at = -1;
          for (int pass = 0; pass <= P.iters; ++pass) {
            float xv[C::KS];
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) xv[dc] = X.z[X.dr * C::KS + dc];
            float d2[C::KB];
#pragma unroll
            for (int k = 0; k < C::KP; ++k) {
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) {
                const float2 e = tsub2(S.pair(k, dc), tf2(xv[dc]));
                acc = tfma2(e, e, acc);
              }
              d2[2 * k] = acc.x;
              d2[2 * k + 1] = acc.y;
            }
            if (C::ODD) {
              float acc = 0.0f;
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) {
                const float e = S.single(dc) - xv[dc];
                acc = fmaf(e, e, acc);
              }
              d2[C::KB - 1] = acc;
            }
            float tot[C::SPL];
            group_point_totals<C>(X, d2, tot);
            float bown[C::SPL], sown[C::SPL];
#pragma unroll
            for (int i = 0; i < C::SPL; ++i) {
              const float w = i == 0 ? wown0 : wown[i];
              const float root = sqrtf(tot[i] + P.epsilon);
              bown[i] = w / root;   // irls.hpp:45-46
              sown[i] = w * root;   // costs.hpp:24-33
            }
            float ball[C::KB], surall[C::KB];
            group_broadcast<C>(X, bown, ball);
            group_broadcast<C>(X, sown, surall);
            float gden = 0.0f, gsur = 0.0f;
#pragma unroll
            for (int m = 0; m < C::KB; ++m) {
              gden += ball[m];
              gsur += surall[m];
            }
            float v[C::KS];
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) {
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int k = 0; k < C::KP; ++k)
                acc = tfma2(make_float2(ball[2 * k], ball[2 * k + 1]), S.pair(k, dc), acc);
              float t2 = acc.x + acc.y;
              if (C::ODD) t2 = fmaf(ball[C::KB - 1], S.single(dc), t2);
              v[dc] = X.active ? t2 : 0.0f;
            }
            if (!X.active) {
              gden = 0.0f;
              gsur = 0.0f;
            }
            if (X.tid == 0) X.flags[pass & 1] = 0;
            __syncthreads();
            irls_reduce<C>(X, v, gden, gsur, [&](int j, float num, float den, float sur) {
              const float xo = X.z[j];
              const float xn = num / den;
              X.a0[j] = xo;  // keep x_pass (the iterate the stop test refers to)
              X.z[j] = xn;
              int f = isfinite(xn) ? 0 : 1;
              if (j == 0) {
                X.scal[16] = sur;
                f |= isfinite(sur) ? 0 : 2;
              }
              if (f) atomicOr(&X.flags[pass & 1], f);
            });
            const int fl = X.flags[pass & 1];
            const float current = X.scal[16];
            if (fl & 2) {  // non-finite surrogate at x_pass (irls.hpp:39, :52)
              fail_iter = pass;
              fail_kind = NLEM_FAIL_IRLS_OBJECTIVE;
              break;
            }
            if (pass >= 1) {
              if (frames && X.tid == 0)
                frames[static_cast<int64_t>(pass - 1) * plane + pix] = clamp_box(X.a0[center], P.range);
              if (previous - current <= P.irls_tol * fabsf(previous)) {  // irls.hpp:58
                stop_at = pass;
                break;
              }
            }
            previous = current;
            if (pass < P.iters && (fl & 1)) {  // non-finite x_{pass+1} (irls.hpp:50)
              fail_iter = pass + 1;
              fail_kind = NLEM_FAIL_IRLS_ITERATE;
              break;
            }
          }
          // the minimiser is x at the stop pass (or x_T); X.a0 holds it, z holds x_{+1}
          if (fail_iter < 0) {
            iters = stop_at > 0 ? stop_at : P.iters;
            if (X.tid < C::D) X.z[X.tid] = X.a0[X.tid];
          }
          __syncthreads();
        }
      }
      if constexpr (C::XW == 4) {
        if (P.solver == NLEM_SOLVER_ADMM) {
          // ---- EM-ADMM sweeps, split p-form.  Between sweeps a lane keeps q_k = s_k p_k - a_k;
          // sweep t forms p_k = q_k + c (c = 2 z_{t-1} - z_{t-2}), the norms, prox scales and g
          // partials (the critical path), folds its warp's group rows, and after one barrier
          // CPT4 threads per coordinate reduce the warp rows and publish z_t and c, with the
          // next q computed between the consensus loads and their reduction.  Same iterates as
          // the p-form (p' = s p + (c - a)) up to FP32 rounding order.
          if (X.tid < C::D) X.cs[(X.tid / C::KS) * C::CSTR + X.tid % C::KS] = X.z[X.tid];
          __syncthreads();
          {
            float lam_own[C::SPL];
#pragma unroll
            for (int i = 0; i < C::SPL; ++i) lam_own[i] = inv_mu * wown[i];
            float2 p2[C::KP][C::KS];  // q between sweeps, p within a sweep
            float p1[C::KS];
#pragma unroll
            for (int qq = 0; qq < C::KP; ++qq)
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) p2[qq][dc] = tsub2(make_float2(0.0f, 0.0f), S.pair(qq, dc));
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) p1[dc] = C::ODD ? -S.single(dc) : 0.0f;
            float* red_row = X.red + (X.grow0 / C::G) * C::GSTR + X.dr * C::KS;
            // c of the coming sweep (this lane's patch row), loaded as soon as it is published
            // (before the flag checks) with 128-bit loads
            float cc[C::CSTR];
            const float4* crow = reinterpret_cast<const float4*>(X.cs + X.dr * C::CSTR);
            auto load_c = [&]() {
#pragma unroll
              for (int i = 0; i < (C::KS + 3) / 4; ++i) {
                const float4 v = crow[i];
                cc[4 * i] = v.x;
                cc[4 * i + 1] = v.y;
                cc[4 * i + 2] = v.z;
                cc[4 * i + 3] = v.w;
              }
            };
            load_c();
            // XW == 4: the consensus thread of coordinate cj (part 0 of CPT4) keeps z_j and a0_j
            const int cj = X.tid / C::CPT4, cpart = X.tid % C::CPT4;
            const bool cfin = cj < C::D && cpart == 0;
            const int cjc = cj < C::D ? cj : 0;
            const int cidx = (cjc / C::KS) * C::CSTR + cjc % C::KS;
            float zreg = X.z[cjc];
            const float a0reg = X.a0[cjc];
            for (int t = 1; t <= P.iters; ++t) {
              WSTAMP(0);
              float nr[C::KB];
              {
#pragma unroll
                for (int qq = 0; qq < C::KP; ++qq) {
                  float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
                  for (int dc = 0; dc < C::KS; ++dc) {
                    p2[qq][dc] = __fadd2_rn(p2[qq][dc], tf2(cc[dc]));
                    acc = tfma2(p2[qq][dc], p2[qq][dc], acc);
                  }
                  nr[2 * qq] = acc.x;
                  nr[2 * qq + 1] = acc.y;
                }
                if (C::ODD) {
                  float acc = 0.0f;
#pragma unroll
                  for (int dc = 0; dc < C::KS; ++dc) {
                    p1[dc] += cc[dc];
                    acc = fmaf(p1[dc], p1[dc], acc);
                  }
                  nr[C::KB - 1] = acc;
                }
              }
              float tot[C::SPL], sown[C::SPL];
              group_point_totals<C>(X, nr, tot);
              int fbits = 0;
#pragma unroll
              for (int i = 0; i < C::SPL; ++i) {
                const float lam = lam_own[i];
                const float s = lam != 0.0f ? fminf(1.0f, lam * rsqrt_ftz(tot[i])) : 0.0f;
                sown[i] = s;
                fbits |= (lam != 0.0f && !isfinite(tot[i])) ? 1 : 0;
                if (static_eq) fbits |= (is_real(X.dr + i * C::G) && s != 1.0f) ? 2 : 0;
              }
              float sall[C::KB];
              group_broadcast<C>(X, sown, sall);
              float2 s2[C::KP];
#pragma unroll
              for (int qq = 0; qq < C::KP; ++qq) s2[qq] = make_float2(sall[2 * qq], sall[2 * qq + 1]);
              const float s1 = C::ODD ? sall[C::KB - 1] : 0.0f;
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) {
                float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int qq = 0; qq < C::KP; ++qq) acc = tfma2(s2[qq], p2[qq][dc], acc);
                float tsum = acc.x + acc.y;
                if (C::ODD) tsum = fmaf(s1, p1[dc], tsum);
                if (X.slot) red_row[dc] = tsum;  // idle slot lanes: s = 0 on finite p -> exact 0
              }
              if (fbits) {  // rare
                atomicOr(&X.flags[t & 1], fbits);
                if (fbits & 1) atomicMin(&X.flags[4], 2 * t + 1);
              }
              WSTAMP(1);
              // next sweep's q = s p - a (overlaps the consensus)
              auto q_update = [&]() {
#pragma unroll
                for (int qq = 0; qq < C::KP; ++qq)
#pragma unroll
                  for (int dc = 0; dc < C::KS; ++dc) {
                    const float2 a = S.pair(qq, dc);
                    p2[qq][dc] = tfma2(s2[qq], p2[qq][dc], make_float2(-a.x, -a.y));
                  }
                if (C::ODD) {
#pragma unroll
                  for (int dc = 0; dc < C::KS; ++dc) p1[dc] = fmaf(s1, p1[dc], -S.single(dc));
                }
              };
              {
                // fold this warp's GPW group rows into its warp row (fixed order)
                __syncwarp();
                if (X.lane < (C::D + 1) / 2) {
                  const float2* g0 =
                      reinterpret_cast<const float2*>(X.red + X.warp * C::GPW * C::GSTR) + X.lane;
                  float2 acc = g0[0];
#pragma unroll
                  for (int i = 1; i < C::GPW; ++i) acc = __fadd2_rn(acc, g0[i * (C::GSTR / 2)]);
                  reinterpret_cast<float2*>(X.wred + X.warp * C::WSTR)[X.lane] = acc;
                }
                __syncthreads();
                {
                  // CPT threads per coordinate; loads first, then the state update, then the
                  // fixed-order reduction (rows part, part + CPT, ...) and the finish
                  constexpr int NPER = C::WARPS / C::CPT4;
                  float lv[NPER];
#pragma unroll
                  for (int i = 0; i < NPER; ++i) lv[i] = X.wred[(cpart + i * C::CPT4) * C::WSTR + cjc];
                  q_update();
#pragma unroll
                  for (int w = 1; w < NPER; w <<= 1)
#pragma unroll
                    for (int i = 0; i + w < NPER; i += 2 * w) lv[i] += lv[i + w];
                  float gsum = lv[0];
#pragma unroll
                  for (int o = 1; o < C::CPT4; o <<= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
                  if (cfin) {
                    const float zo = zreg;
                    const float zn = clamp_box(fmaf(-gsum, inv_n, zo), P.range);
                    int f = isfinite(zn) ? 0 : 4;
                    if (static_eq) f |= (zn != a0reg) ? 8 : 0;
                    zreg = zn;
                    X.z[cj] = zn;
                    X.cs[cidx] = 2.0f * zn - zo;
                    if (f) {
                      atomicOr(&X.flags[t & 1], f);
                      if (f & 4) atomicMin(&X.flags[4], 2 * t);
                    }
                    if (cj == 0) X.flags[(t + 1) & 1] = 0;
                  }
                  WSTAMP(2);
                  __syncthreads();
                }
              }
              WSTAMP(3);
              load_c();
#ifdef NLEM_PHASE_PROFILE
              ++X.dbg_it;
#endif
              {
                // failures are recorded as the first failing sweep (flags[4]) and decoded after
                // the loop: no per-sweep flag read or divergent branch on the critical path; the
                // flag word is read only when the exact-stop test is possible (constant footprint)
                if (frames != nullptr) {
                  if (X.tid == 0) frames[static_cast<int64_t>(t - 1) * plane + pix] = X.z[center];
                }
                if (static_eq) {
                  const int fl = X.flags[t & 1];
                  if (!(fl & (4 | 1 | 2 | 8)) && X.flags[4] == 0x7fffffff) {  // residual exactly 0
                    iters = t;
                    break;
                  }
                }
              }
            }
            {
              // decode the first failure: non-finite z at sweep t -> t; a non-finite norm at
              // sweep t (multiplier blow-up in t - 1) -> t - 1, or t for t = 1
              const int fw = X.flags[4];
              if (fw != 0x7fffffff) {
                const int tf = fw >> 1;
                fail_iter = !(fw & 1) || tf == 1 ? tf : tf - 1;
                fail_kind = NLEM_FAIL_ADMM_ITERATE;
              }
            }
          }
        }
      } else if (P.solver == NLEM_SOLVER_ADMM) {
        // ---- EM-ADMM sweeps in p-form (see solver_generic.cuh)
        float lam_own[C::SPL];
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) lam_own[i] = inv_mu * wown[i];
        float2 p2[C::KP][C::KS];
        float p1[C::KS];
        float2 s2[C::KP];
        float s1 = 0.0f;
#pragma unroll
        for (int qq = 0; qq < C::KP; ++qq) {
          s2[qq] = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) p2[qq][dc] = make_float2(0.0f, 0.0f);
        }
#pragma unroll
        for (int dc = 0; dc < C::KS; ++dc) p1[dc] = 0.0f;
        // c of the first sweep = z0 (p = 0*p + z0 - a)
        if (X.tid < C::D) X.c2[X.tid] = tf2(X.z[X.tid]);
        __syncthreads();
        for (int t = 1; t <= P.iters; ++t) {
          PHASE(0);
          WSTAMP(0);
          // (U) p' = s p + (c - a); per-point norm partials
          float nr[C::KB];
          {
            float2 cc[C::KS];
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) cc[dc] = X.c2[X.dr * C::KS + dc];
#pragma unroll
            for (int qq = 0; qq < C::KP; ++qq) {
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) {
                const float2 ca = tsub2(cc[dc], S.pair(qq, dc));
                p2[qq][dc] = tfma2(s2[qq], p2[qq][dc], ca);
                acc = tfma2(p2[qq][dc], p2[qq][dc], acc);
              }
              nr[2 * qq] = acc.x;
              nr[2 * qq + 1] = acc.y;
            }
            if (C::ODD) {
              float acc = 0.0f;
#pragma unroll
              for (int dc = 0; dc < C::KS; ++dc) {
                p1[dc] = fmaf(s1, p1[dc], cc[dc].x - S.single(dc));
                acc = fmaf(p1[dc], p1[dc], acc);
              }
              nr[C::KB - 1] = acc;
            }
          }
          // (R) group totals -> prox scales -> broadcast
          PHASE(1);
          float tot[C::SPL], sown[C::SPL];
          group_point_totals<C>(X, nr, tot);
          PHASE(2);
          int fbits = 0;
#pragma unroll
          for (int i = 0; i < C::SPL; ++i) {
            const float lam = lam_own[i];
            const float s = lam != 0.0f ? fminf(1.0f, lam * rsqrt_ftz(tot[i])) : 0.0f;
            sown[i] = s;
            fbits |= (lam != 0.0f && !isfinite(tot[i])) ? 1 : 0;
            if (static_eq) fbits |= (is_real(X.dr + i * C::G) && s != 1.0f) ? 2 : 0;
          }
          float sall[C::KB];
          group_broadcast<C>(X, sown, sall);
#pragma unroll
          for (int qq = 0; qq < C::KP; ++qq) s2[qq] = make_float2(sall[2 * qq], sall[2 * qq + 1]);
          if (C::ODD) s1 = sall[C::KB - 1];
          PHASE(3);
          // (G) g partials per coordinate
          float v[C::KS];
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) {
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int qq = 0; qq < C::KP; ++qq) acc = tfma2(s2[qq], p2[qq][dc], acc);
            float tsum = acc.x + acc.y;
            if (C::ODD) tsum = fmaf(s1, p1[dc], tsum);
            v[dc] = X.active ? tsum : 0.0f;
          }
          fbits = __reduce_or_sync(0xffffffffu, fbits);
          if (X.lane == 0 && fbits) atomicOr(&X.flags[t & 1], fbits);
          PHASE(4);
          // consensus z_t = P_C(z - g/n), c = 2 z_t - z  (admm.hpp:59-65 in p-form)
          reduce_coordinates<C>(X, v, [&](int j, float gsum) {
            const float zo = X.z[j];
            const float zn = clamp_box(fmaf(-gsum, inv_n, zo), P.range);
            int f = isfinite(zn) ? 0 : 4;
            if (static_eq) f |= (zn != X.a0[j]) ? 8 : 0;  // exact-stop test only if possible
            X.z[j] = zn;
            X.c2[j] = tf2(2.0f * zn - zo);
            if (f) atomicOr(&X.flags[t & 1], f);  // rare: non-finite, or a constant footprint
            if (j == 0) X.flags[(t + 1) & 1] = 0;  // all reads of sweep t-1's word are done
          });
          const int fl = X.flags[t & 1];
          PHASE(5);
#ifdef NLEM_PHASE_PROFILE
          ++X.dbg_it;
#endif
          if (fl & (4 | 1)) {
            fail_iter = (fl & 4) || t == 1 ? t : t - 1;
            fail_kind = NLEM_FAIL_ADMM_ITERATE;
            break;
          }
          if (frames && X.tid == 0)
            frames[static_cast<int64_t>(t - 1) * plane + pix] = X.z[center];
          if (static_eq && !(fl & 2) && !(fl & 8)) {  // residual exactly 0 (admm.hpp:77)
            iters = t;
            break;
          }
        }
      }
      SSTAMP(6);
#ifdef NLEM_PHASE_PROFILE
      ++X.dbg_px;
#endif
      if (X.tid == 0) {
        if (fail_iter >= 0) {
          record_failure(fail, r * cols + c, fail_iter, fail_kind);
        } else {
          float v = X.z[center];
          if (P.solver != NLEM_SOLVER_ADMM) v = clamp_box(v, P.range);  // NlmOnly (nlem.cpp:26-31)
          out[pix] = v;
          if (frames) {
            const int from = P.solver == NLEM_SOLVER_NLM_ONLY ? 0 : iters;
            for (int t = from; t < P.iters; ++t) frames[static_cast<int64_t>(t) * plane + pix] = v;
          }
        }
      }
      __syncthreads();
    }
    ch = next_chunk();
    chunk_parity ^= 1;
  }
}

namespace {

template <class C>
cudaError_t launch_tile(const NlemLaunch& L, cudaStream_t stream, const int* list = nullptr,
                        const int* list_count = nullptr) {
  const size_t smem = TileSmem<C>::TOTAL * sizeof(float);
  auto kfn = nlem_pixels_tile<C>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t pixels = L.out_rows * L.cols;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, C::THREADS, smem);
  int64_t ctas = int64_t(device_caps().sms) * std::max(per_sm, 1);
  const int chunk = list ? 1 : static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, pixels / (ctas * 4))));
  ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, (pixels + chunk - 1) / chunk));
  int* counter = nullptr;  // dynamic chunk counter (stream-ordered scratch)
  e = cudaMallocAsync(&counter, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e == cudaSuccess) {
    kfn<<<static_cast<unsigned>(ctas), C::THREADS, smem, stream>>>(
        L.pad, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out, L.frames, counter,
        chunk, L.fail, list, list_count);
    e = cudaGetLastError();
  }
  const cudaError_t ef = cudaFreeAsync(counter, stream);
  return e != cudaSuccess ? e : ef;
}

}  // namespace

#ifdef NLEM_PHASE_PROFILE
}  // namespace nlemk
extern "C" int nlem_debug_phase_times(long long* out /* [2][64][16] */) {
  return cudaMemcpyFromSymbol(out, nlemk::g_phase, sizeof(nlemk::g_phase)) == cudaSuccess ? 0 : 1;
}
extern "C" int nlem_debug_setup_times(long long* out /* [64][8] */) {
  return cudaMemcpyFromSymbol(out, nlemk::g_setup, sizeof(nlemk::g_setup)) == cudaSuccess ? 0 : 1;
}
extern "C" int nlem_debug_warp_times(long long* out /* [32][64][4] */) {
  return cudaMemcpyFromSymbol(out, nlemk::g_warp, sizeof(nlemk::g_warp)) == cudaSuccess ? 0 : 1;
}
namespace nlemk {
#endif

bool nlem_tile_supported(const NlemLaunch& L) {
  // smaller (odd) windows run masked inside the kernel's grid
  return (L.P.patch == 7 || L.P.patch == 5 || L.P.patch == 3) && L.P.search <= 21;
}

int nlem_tile_grid(const NlemLaunch& L) {  // side of the grid the serving instantiation uses
  return L.P.patch == 7 || L.P.search > 11 ? 21 : 11;
}

cudaError_t launch_nlem_tile_list(const NlemLaunch& L, const int* list, const int* list_count,
                                  cudaStream_t stream) {
  const bool big = nlem_tile_grid(L) == 21;
  if (L.P.patch == 7) return launch_tile<TileK7S21>(L, stream, list, list_count);
  if (L.P.patch == 5)
    return big ? launch_tile<TileK5S21>(L, stream, list, list_count)
               : launch_tile<TileK5S11>(L, stream, list, list_count);
  return big ? launch_tile<TileK3S21>(L, stream, list, list_count)
             : launch_tile<TileK3S11>(L, stream, list, list_count);
}

cudaError_t launch_nlem_tile(const NlemLaunch& L, cudaStream_t stream) {
  return launch_nlem_tile_list(L, nullptr, nullptr, stream);
}

}  // namespace nlemk
