// NLEM sliding-window kernel, two window segments per lane (configs 2, 3; k = 7, S = 21).
//
// Same algorithm and data flow as kernels_nlem_tile.cu (read that header first): the 21 x 21
// window grid of a pixel is cut into 63 segments of 7 consecutive grid points; a lane owns
// NSEG = 2 segments x one patch row (2 x 7 points x 7 coordinates = 98 elements of the p-form
// iterate in registers, plus the 2 x 13 image values those elements read).  Doubling the
// elements per lane halves every per-element share of the per-sweep fixed costs that the
// one-segment kernel was bound by (profiles/r1_tile_phase_times.txt): shared-memory
// wavefronts for c, the norm transpose, the prox-scale broadcast and the partial-g writes,
// plus the instruction overhead around them.  32 groups of 7 lanes = 8 warps per pixel.
#include <algorithm>

#include "launch.h"
#include "solver_generic.cuh"

namespace nlemk {

template <int KS_, int SW_, int KB_, int NSEG_>
struct Seg2Cfg {
  static constexpr int KS = KS_, SW = SW_, KB = KB_, NSEG = NSEG_;
  static constexpr int D = KS * KS;
  static constexpr int G = KS;                          // lanes per group (patch rows)
  static constexpr int GPW = 32 / G;                    // groups per warp
  static constexpr int NBLK = SW / KB;                  // segments per grid row
  static constexpr int NSEGS = SW * NBLK;               // segments per pixel
  static constexpr int NGROUPS = (NSEGS + NSEG - 1) / NSEG;
  static constexpr int WARPS = (NGROUPS + GPW - 1) / GPW;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int PL = NSEG * KB;                  // points per lane
  static constexpr int KP = KB / 2;
  static constexpr bool ODD = (KB % 2) != 0;
  static constexpr int SEG = KB + KS - 1;
  static constexpr int TH = SW + KS - 1;
  static constexpr int TWS = (TH + 4) & ~1;
  static constexpr int NE = ((KP - 1 + (KS - 1) / 2) > ((SEG - 1) / 2) ? (KP - 1 + (KS - 1) / 2)
                                                                        : ((SEG - 1) / 2)) + 1;
  static constexpr int NO = KP - 1 + (KS - 2) / 2 + 1;
  static constexpr int PLP = (PL + 3) & ~3;             // padded per-lane point row
  static constexpr int SPL = (PL + G - 1) / G;          // points whose scale a lane computes
  static constexpr int CPT = THREADS >= 8 * D ? 8 : THREADS >= 4 * D ? 4 : THREADS >= 2 * D ? 2 : 1;
  static constexpr int GSTR = 52;                       // group stride of g partials (D=49)
  static_assert(SW % KB == 0 && D == 49, "k = 7 only");
};

using Seg2K7 = Seg2Cfg<7, 21, 7, 2>;

template <class C>
struct Seg2Smem {
  static constexpr int T = C::TH * C::TWS;
  static constexpr int ROWS = C::NGROUPS * C::G + 40;
  static constexpr int NB = ROWS * C::PLP;
  static constexpr int RED = (C::NGROUPS + 8) * C::GSTR;
  static constexpr int TOTAL = 2 * T + NB + RED + 2 * C::D + 2 * C::D + 64;
};

__device__ __forceinline__ float2 s2f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 s2sub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 s2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float s2rsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <class C>
struct Seg2Vals {
  float2 E[C::NE];
  float2 O[C::NO];
  __device__ __forceinline__ float2 pair(int q, int dc) const {
    return (dc & 1) ? O[q + (dc - 1) / 2] : E[q + dc / 2];
  }
  __device__ __forceinline__ float single(int dc) const {
    const int x = C::KB - 1 + dc;
    return (x & 1) ? E[x / 2].y : E[x / 2].x;
  }
};

template <class C>
struct Seg2Ctx {
  float *T0, *T1, *nbuf, *red;
  float2* c2;
  float *z, *a0, *scal;
  int* flags;
  int tid, warp, lane, q, dr, base, grow0;
  bool active;
  int gr[C::NSEG], gc0[C::NSEG];
  bool segv[C::NSEG];

  __device__ void carve(float* smem) {
    T0 = smem;
    T1 = T0 + Seg2Smem<C>::T;
    nbuf = T1 + Seg2Smem<C>::T;
    red = nbuf + Seg2Smem<C>::NB;
    c2 = reinterpret_cast<float2*>(red + Seg2Smem<C>::RED);
    z = reinterpret_cast<float*>(c2 + C::D);
    a0 = z + C::D;
    flags = reinterpret_cast<int*>(a0 + C::D);
    scal = reinterpret_cast<float*>(flags + 8);
    tid = threadIdx.x;
    warp = tid >> 5;
    lane = tid & 31;
    const int ql = lane / C::G;
    dr = lane - ql * C::G;
    base = ql * C::G;
    q = warp * C::GPW + ql;
    active = ql < C::GPW && q < C::NGROUPS;
    grow0 = active ? q * C::G : C::NGROUPS * C::G + base;
#pragma unroll
    for (int sg = 0; sg < C::NSEG; ++sg) {
      const int si = (active ? q : 0) * C::NSEG + sg;
      segv[sg] = active && si < C::NSEGS;
      const int sic = si < C::NSEGS ? si : 0;
      gr[sg] = sic / C::NBLK;
      gc0[sg] = (sic % C::NBLK) * C::KB;
    }
  }
};

template <class C>
__device__ __forceinline__ float seg2_tree(const float* col, int stride) {
  float v[C::G];
#pragma unroll
  for (int r = 0; r < C::G; ++r) v[r] = col[r * stride];
#pragma unroll
  for (int w = 1; w < C::G; w <<= 1)
#pragma unroll
    for (int r = 0; r + w < C::G; r += 2 * w) v[r] += v[r + w];
  return v[0];
}

// per-point partials v[PL] -> this lane's SPL point totals (points m = dr + i*G)
template <class C>
__device__ __forceinline__ void seg2_point_totals(Seg2Ctx<C>& X, const float (&v)[C::PL],
                                                  float (&tot)[C::SPL]) {
  float* row = X.nbuf + (X.grow0 + X.dr) * C::PLP;
#pragma unroll
  for (int m = 0; m < C::PL; ++m) row[m] = v[m];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < C::SPL; ++i) {
    const int m = X.dr + i * C::G;
    tot[i] = m < C::PL ? seg2_tree<C>(X.nbuf + X.grow0 * C::PLP + (m < C::PL ? m : 0), C::PLP) : 0.0f;
  }
  __syncwarp();
}

template <class C>
__device__ __forceinline__ void seg2_broadcast(const Seg2Ctx<C>& X, const float (&own)[C::SPL],
                                               float (&all)[C::PL]) {
#pragma unroll
  for (int m = 0; m < C::PL; ++m) {
    float v = own[0];
#pragma unroll
    for (int i = 1; i < C::SPL; ++i)
      if (m / C::G == i) v = own[i];
    all[m] = __shfl_sync(0xffffffffu, v, X.base + m % C::G);
  }
}

template <class C, class Finish>
__device__ __forceinline__ void seg2_reduce(Seg2Ctx<C>& X, const float (&v)[C::KS], Finish finish) {
  {
    float* row = X.red + (X.grow0 / C::G) * C::GSTR + X.dr * C::KS;
#pragma unroll
    for (int dc = 0; dc < C::KS; ++dc) row[dc] = v[dc];
  }
  __syncthreads();
  const int j = X.tid / C::CPT, part = X.tid % C::CPT;
  float s = 0.0f;
  if (j < C::D) {
    const float* col = X.red + part * C::GSTR + j;
    constexpr int NPER = (C::NGROUPS + C::CPT - 1) / C::CPT;
    float w[NPER];
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      w[i] = (part + i * C::CPT < C::NGROUPS) ? col[i * C::CPT * C::GSTR] : 0.0f;
#pragma unroll
    for (int st = 1; st < NPER; st <<= 1)
#pragma unroll
      for (int i = 0; i + st < NPER; i += 2 * st) w[i] += w[i + st];
    s = w[0];
  }
#pragma unroll
  for (int o = 1; o < C::CPT; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (j < C::D && part == 0) finish(j, s);
  __syncthreads();
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
nlem_pixels_seg2(const float* __restrict__ pad, int64_t pad_cols, int64_t rows, int64_t cols,
                 int64_t out_row0, int64_t out_rows, NlemDevParams P, float* out, float* frames,
                 int chunk, FailureSlot* fail) {
  extern __shared__ __align__(16) float smem[];
  Seg2Ctx<C> X;
  X.carve(smem);
  constexpr int hs = C::SW / 2;
  constexpr int center = C::D / 2;
  const int64_t plane = out_rows * cols;
  const int64_t nchunks = (plane + chunk - 1) / chunk;
  const float inv_mu = 1.0f / P.mu;
  int offE[C::NSEG], offO[C::NSEG];
  bool t1E[C::NSEG];
#pragma unroll
  for (int sg = 0; sg < C::NSEG; ++sg) {
    const int trow = X.gr[sg] + X.dr;
    const bool even = (X.gc0[sg] & 1) == 0;
    offE[sg] = trow * C::TWS + (even ? X.gc0[sg] : X.gc0[sg] - 1);
    offO[sg] = trow * C::TWS + (even ? X.gc0[sg] : X.gc0[sg] + 1);
    t1E[sg] = !even;
  }
  for (int e = X.tid; e < 2 * Seg2Smem<C>::T; e += C::THREADS) X.T0[e] = 0.0f;
  __syncthreads();

  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t pix_end = (ch + 1) * chunk < plane ? (ch + 1) * chunk : plane;
    for (int64_t pix = ch * chunk; pix < pix_end; ++pix) {
      const int64_t r = out_row0 + pix / cols, c = pix % cols;
      const int gr0 = r < hs ? static_cast<int>(hs - r) : 0;
      const int gr1 = rows - 1 - r < hs ? static_cast<int>(hs + (rows - 1 - r)) : C::SW - 1;
      const int gc0w = c < hs ? static_cast<int>(hs - c) : 0;
      const int gc1w = cols - 1 - c < hs ? static_cast<int>(hs + (cols - 1 - c)) : C::SW - 1;
      const int n = (gr1 - gr0 + 1) * (gc1w - gc0w + 1);
      const float inv_n = 1.0f / static_cast<float>(n);
      const float* src = pad + (r - out_row0) * pad_cols + c;
      for (int e = X.tid; e < C::TH * C::TH; e += C::THREADS) {
        const int tr = e / C::TH, tc = e - tr * C::TH;
        const float v = __ldg(src + tr * pad_cols + tc);
        X.T0[tr * C::TWS + tc] = v;
        if (tc > 0) X.T1[tr * C::TWS + tc - 1] = v;
      }
      __syncthreads();
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
      }
      Seg2Vals<C> S[C::NSEG];
#pragma unroll
      for (int sg = 0; sg < C::NSEG; ++sg) {
        const float2* pE = reinterpret_cast<const float2*>((t1E[sg] ? X.T1 : X.T0) + offE[sg]);
        const float2* pO = reinterpret_cast<const float2*>((t1E[sg] ? X.T0 : X.T1) + offO[sg]);
#pragma unroll
        for (int i = 0; i < C::NE; ++i) S[sg].E[i] = pE[i];
#pragma unroll
        for (int i = 0; i < C::NO; ++i) S[sg].O[i] = pO[i];
      }
      const bool static_eq = !__syncthreads_or(neq);
      auto is_real = [&](int m) {
        const int sg = m / C::KB, mm = m - sg * C::KB;
        bool rr = false;
#pragma unroll
        for (int k = 0; k < C::NSEG; ++k)
          if (k == sg)
            rr = X.segv[k] && X.gr[k] >= gr0 && X.gr[k] <= gr1 && X.gc0[k] + mm >= gc0w &&
                 X.gc0[k] + mm <= gc1w;
        return rr && m < C::PL;
      };
      // ---- weights
      float wown[C::SPL];
      {
        float sv[C::KS];
#pragma unroll
        for (int dc = 0; dc < C::KS; ++dc) sv[dc] = X.T0[(hs + X.dr) * C::TWS + hs + dc];
        float d2[C::PL];
#pragma unroll
        for (int sg = 0; sg < C::NSEG; ++sg) {
#pragma unroll
          for (int qq = 0; qq < C::KP; ++qq) {
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) {
              const float2 e = s2sub(S[sg].pair(qq, dc), s2f2(sv[dc]));
              acc = s2fma(e, e, acc);
            }
            d2[sg * C::KB + 2 * qq] = acc.x;
            d2[sg * C::KB + 2 * qq + 1] = acc.y;
          }
          if (C::ODD) {
            float acc = 0.0f;
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) {
              const float e = S[sg].single(dc) - sv[dc];
              acc = fmaf(e, e, acc);
            }
            d2[sg * C::KB + C::KB - 1] = acc;
          }
        }
        float tot[C::SPL];
        seg2_point_totals<C>(X, d2, tot);
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) wown[i] = is_real(X.dr + i * C::G) ? expf(-tot[i] * P.inv_h2) : 0.0f;
      }
      float wall[C::PL];
      seg2_broadcast<C>(X, wown, wall);
      const bool nlm_init = P.solver == NLEM_SOLVER_NLM_ONLY || P.init_mode == NLEM_INIT_NLM_PATCH;
      if (nlm_init) {
        float wsum = 0.0f;
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) wsum += wown[i];
        wsum = warp_sum(X.active ? wsum : 0.0f);
        if (X.lane == 0) X.scal[X.warp] = wsum;
        __syncthreads();
        float W = 0.0f;
#pragma unroll
        for (int w = 0; w < C::WARPS; ++w) W += X.scal[w];
        const bool ratio = P.nlm_ratio != 0;
        float v[C::KS];
#pragma unroll
        for (int dc = 0; dc < C::KS; ++dc) v[dc] = 0.0f;
#pragma unroll
        for (int sg = 0; sg < C::NSEG; ++sg) {
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) {
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int qq = 0; qq < C::KP; ++qq) {
              const float c0 = wall[sg * C::KB + 2 * qq], c1 = wall[sg * C::KB + 2 * qq + 1];
              acc = s2fma(ratio ? make_float2(c0, c1) : make_float2(c0 / W, c1 / W), S[sg].pair(qq, dc), acc);
            }
            float t = acc.x + acc.y;
            if (C::ODD) {
              const float cl = wall[sg * C::KB + C::KB - 1];
              t = fmaf(ratio ? cl : cl / W, S[sg].single(dc), t);
            }
            v[dc] += t;
          }
        }
        seg2_reduce<C>(X, v, [&](int j, float tsum) { X.z[j] = ratio ? tsum / W : tsum; });
      } else {
        if (X.tid < C::D) {
          const int jr = X.tid / C::KS, jc = X.tid - jr * C::KS;
          X.z[X.tid] = X.T0[(hs + jr) * C::TWS + hs + jc];
        }
        __syncthreads();
      }

      int iters = P.iters, fail_iter = -1, fail_kind = 0;
      if (P.solver == NLEM_SOLVER_ADMM) {
        float lam_own[C::SPL];
#pragma unroll
        for (int i = 0; i < C::SPL; ++i) lam_own[i] = inv_mu * wown[i];
        float2 p2[C::NSEG][C::KP][C::KS];
        float p1[C::NSEG][C::KS];
        float2 s2[C::NSEG][C::KP];
        float s1[C::NSEG];
#pragma unroll
        for (int sg = 0; sg < C::NSEG; ++sg) {
          s1[sg] = 0.0f;
#pragma unroll
          for (int qq = 0; qq < C::KP; ++qq) {
            s2[sg][qq] = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) p2[sg][qq][dc] = make_float2(0.0f, 0.0f);
          }
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) p1[sg][dc] = 0.0f;
        }
        if (X.tid < C::D) X.c2[X.tid] = s2f2(X.z[X.tid]);
        __syncthreads();
        for (int t = 1; t <= P.iters; ++t) {
          float nr[C::PL];
          {
            float2 cc[C::KS];
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) cc[dc] = X.c2[X.dr * C::KS + dc];
#pragma unroll
            for (int sg = 0; sg < C::NSEG; ++sg) {
#pragma unroll
              for (int qq = 0; qq < C::KP; ++qq) {
                float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int dc = 0; dc < C::KS; ++dc) {
                  const float2 ca = s2sub(cc[dc], S[sg].pair(qq, dc));
                  p2[sg][qq][dc] = s2fma(s2[sg][qq], p2[sg][qq][dc], ca);
                  acc = s2fma(p2[sg][qq][dc], p2[sg][qq][dc], acc);
                }
                nr[sg * C::KB + 2 * qq] = acc.x;
                nr[sg * C::KB + 2 * qq + 1] = acc.y;
              }
              if (C::ODD) {
                float acc = 0.0f;
#pragma unroll
                for (int dc = 0; dc < C::KS; ++dc) {
                  p1[sg][dc] = fmaf(s1[sg], p1[sg][dc], cc[dc].x - S[sg].single(dc));
                  acc = fmaf(p1[sg][dc], p1[sg][dc], acc);
                }
                nr[sg * C::KB + C::KB - 1] = acc;
              }
            }
          }
          float tot[C::SPL], sown[C::SPL];
          seg2_point_totals<C>(X, nr, tot);
          int fbits = 0;
#pragma unroll
          for (int i = 0; i < C::SPL; ++i) {
            const float lam = lam_own[i];
            const float s = lam != 0.0f ? fminf(1.0f, lam * s2rsqrt(tot[i])) : 0.0f;
            sown[i] = s;
            fbits |= (lam != 0.0f && !isfinite(tot[i])) ? 1 : 0;
            if (static_eq) fbits |= (is_real(X.dr + i * C::G) && s != 1.0f) ? 2 : 0;
          }
          float sall[C::PL];
          seg2_broadcast<C>(X, sown, sall);
          float v[C::KS];
#pragma unroll
          for (int dc = 0; dc < C::KS; ++dc) v[dc] = 0.0f;
#pragma unroll
          for (int sg = 0; sg < C::NSEG; ++sg) {
#pragma unroll
            for (int qq = 0; qq < C::KP; ++qq)
              s2[sg][qq] = make_float2(sall[sg * C::KB + 2 * qq], sall[sg * C::KB + 2 * qq + 1]);
            if (C::ODD) s1[sg] = sall[sg * C::KB + C::KB - 1];
#pragma unroll
            for (int dc = 0; dc < C::KS; ++dc) {
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int qq = 0; qq < C::KP; ++qq) acc = s2fma(s2[sg][qq], p2[sg][qq][dc], acc);
              float tsum = acc.x + acc.y;
              if (C::ODD) tsum = fmaf(s1[sg], p1[sg][dc], tsum);
              v[dc] += tsum;
            }
          }
          fbits = __reduce_or_sync(0xffffffffu, fbits);
          if (X.lane == 0 && fbits) atomicOr(&X.flags[t & 1], fbits);
          seg2_reduce<C>(X, v, [&](int j, float gsum) {
            const float zo = X.z[j];
            const float zn = clamp_box(fmaf(-gsum, inv_n, zo), P.range);
            int f = isfinite(zn) ? 0 : 4;
            if (static_eq) f |= (zn != X.a0[j]) ? 8 : 0;
            X.z[j] = zn;
            X.c2[j] = s2f2(2.0f * zn - zo);
            if (f) atomicOr(&X.flags[t & 1], f);
            if (j == 0) X.flags[(t + 1) & 1] = 0;
          });
          const int fl = X.flags[t & 1];
          if (fl & (4 | 1)) {
            fail_iter = (fl & 4) || t == 1 ? t : t - 1;
            fail_kind = NLEM_FAIL_ADMM_ITERATE;
            break;
          }
          if (frames && X.tid == 0) frames[static_cast<int64_t>(t - 1) * plane + pix] = X.z[center];
          if (static_eq && !(fl & 2) && !(fl & 8)) {
            iters = t;
            break;
          }
        }
      }
      if (X.tid == 0) {
        if (fail_iter >= 0) {
          record_failure(fail, r * cols + c, fail_iter, fail_kind);
        } else {
          float v = X.z[center];
          if (P.solver != NLEM_SOLVER_ADMM) v = clamp_box(v, P.range);
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

bool nlem_seg2_supported(const NlemLaunch& L) {
  return L.P.solver != NLEM_SOLVER_IRLS && L.P.patch == 7 && L.P.search == 21;
}

cudaError_t launch_nlem_seg2(const NlemLaunch& L, cudaStream_t stream) {
  using C = Seg2K7;
  const size_t smem = Seg2Smem<C>::TOTAL * sizeof(float);
  auto kfn = nlem_pixels_seg2<C>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, C::THREADS, smem);
  const int64_t pixels = L.out_rows * L.cols;
  const int64_t ctas = int64_t(device_caps().sms) * std::max(per_sm, 1);
  const int chunk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, pixels / (ctas * 4))));
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ctas, (pixels + chunk - 1) / chunk));
  kfn<<<static_cast<unsigned>(grid), C::THREADS, smem, stream>>>(
      L.pad, L.pad_cols, L.rows, L.cols, L.out_row0, L.out_rows, L.P, L.out, L.frames, chunk, L.fail);
  return cudaGetLastError();
}

}  // namespace nlemk
