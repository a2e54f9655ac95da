// Generic EM-ADMM and IRLS per-problem solvers: one CTA (kGenThreads threads) per
// problem, warp-per-point passes, any (n, d) with d <= 32*JPL.  State lives in the
// caller-provided buffers (shared memory when it fits, else a global scratch slab).
//
// The ADMM recursion runs in the algebraic "p-form" of Algorithm 1
// (proj/include/nlem/admm.hpp:49-78; derivation SURVEY.md §8a row 3):
//   p_k = z - y_k/mu - a_k,  s_k = prox_scale(w_k/mu, ||p_k||^2)
//   z'  = P_C(z - (1/n) sum_k s_k p_k)                     (admm.hpp:53-59)
//   p_k'= (2z' - z) - a_k + s_k p_k                        (admm.hpp:61-65)
//   x_k - z' = (a_k - z') + (1 - s_k) p_k                  (primal residual terms)
// which needs one n x d state array instead of the reference's two (x, y) and
// four FP32 ops per element per sweep instead of ~12.  n == 1 problems run the
// reference form verbatim so the documented single-point early exits
// (proj/tests/unit/test_solvers.cpp:63-110) reproduce exactly.
#pragma once

#include "common.cuh"

namespace nlemk {

constexpr int kGenThreads = 256;
constexpr int kGenWarps = kGenThreads / kWarpSize;


// Block-shared scratch for one problem.
struct GenWork {
  float* s;      // [n]  prox scales s_k of the current sweep
  float* wts;    // [n]  weights (NLEM: computed in-kernel; batched: copied)
  float* gpart;  // [kGenWarps][dstride] per-warp partial sums
  float* z;      // [d]
  float* zprev;  // [d]
  float* red;    // [4 * kGenWarps]
  int dstride;
};

__host__ __device__ inline size_t gen_work_floats(int n, int d) {
  const int ds = (d + 3) & ~3;
  return static_cast<size_t>(2 * n + kGenWarps * ds + 2 * ds + 4 * kGenWarps + 8);
}

__device__ inline GenWork carve_gen_work(float* base, int n, int d) {
  GenWork W;
  W.dstride = (d + 3) & ~3;
  W.s = base;
  W.wts = W.s + n;
  W.gpart = W.wts + n;
  W.z = W.gpart + kGenWarps * W.dstride;
  W.zprev = W.z + W.dstride;
  W.red = W.zprev + W.dstride;
  return W;
}

struct SolveStatus {
  int iterations;
  int fail_iter;  // -1 none
  int fail_kind;
};

struct NoSnapshot {
  __device__ void operator()(int, const float*) const {}
};

// Block-wide em_cost(z) = sum_k w_k ||z - a_k|| (proj/include/nlem/costs.hpp:13-20),
// fixed reduction order (per warp sequential over its points, then warps 0..7).
template <int JPL>
__device__ float block_em_cost(const float* a, const float* w, int n, int d, const float* z,
                               float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc = 0.0f;
  for (int k = warp; k < n; k += kGenWarps) {
    const float* ak = a + static_cast<size_t>(k) * d;
    float s2 = 0.0f;
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) {
        const float t = z[j] - ak[j];
        s2 = fmaf(t, t, s2);
      }
    }
    s2 = warp_sum(s2);
    acc = fmaf(w[k], sqrtf(s2), acc);
  }
  __syncthreads();
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int i = 0; i < kGenWarps; ++i) tot += red[i];
  __syncthreads();
  return tot;
}

// Problems at or below this dimension (and every n <= 2 problem) run the reference
// form of the sweep verbatim: there the primal residual can hit exactly zero in
// finitely many sweeps (1-D medians, single points: proj/tests/unit/test_solvers.cpp
// :63-151; two points: the duals stay antisymmetric, the iterates stay on the line through
// the points and x_1 == x_2 == z happens exactly, e.g. at sweep 3 for a random pair in d = 49,
// in FP64 and FP32 alike), and only the reference's own arithmetic reproduces the exact stop.
constexpr int kRefFormMaxDim = 16;

__host__ __device__ inline bool use_ref_form(int n, int d) { return n <= 2 || d <= kRefFormMaxDim; }

// floats of solver state per problem (p-form: p; reference form: x and y)
__host__ __device__ inline size_t admm_state_floats(int n, int d, bool force_ref = false) {
  return static_cast<size_t>(n) * d * (force_ref || use_ref_form(n, d) ? 2 : 1);
}

// Reference-form block sweep (admm.hpp:49-78 in float): state y (multipliers) and x
// (local copies), warp per point, per-warp then cross-warp reductions.
template <int JPL, class OnIter>
__device__ SolveStatus admm_solve_refform(const float* a, const float* w, float* xs, float* ys,
                                          int n, int d, GenWork& W, nlem_box box, float mu, int T,
                                          float tol, float* trace_obj, float* trace_res,
                                          OnIter on_iter) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float inv_mu = 1.0f / mu;
  const float nf = static_cast<float>(n);
  const bool want_obj = trace_obj != nullptr;
  SolveStatus st{T, -1, 0};
  for (size_t e = tid; e < static_cast<size_t>(n) * d; e += kGenThreads) ys[e] = 0.0f;  // admm.hpp:41
  __syncthreads();
  for (int t = 1; t <= T; ++t) {
    float zc[JPL], racc[JPL];
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      zc[q] = j < d ? W.z[j] : 0.0f;
      racc[q] = 0.0f;
    }
    for (int k = warp; k < n; k += kGenWarps) {  // admm.hpp:53-57
      const float* ak = a + static_cast<size_t>(k) * d;
      float* yk = ys + static_cast<size_t>(k) * d;
      float* xk = xs + static_cast<size_t>(k) * d;
      float v[JPL], pull[JPL], yv[JPL], av[JPL];
      float d2 = 0.0f;
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        yv[q] = j < d ? yk[j] : 0.0f;
        av[q] = j < d ? ak[j] : 0.0f;
        v[q] = zc[q] - inv_mu * yv[q];
        pull[q] = v[q] - av[q];
        if (j < d) d2 = fmaf(pull[q], pull[q], d2);
      }
      const float lam = inv_mu * w[k];
      const float dist = sqrtf(warp_sum(d2));
      const float f = lam / dist;
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        const float x = lam == 0.0f ? v[q] : (dist <= lam ? av[q] : v[q] - f * pull[q]);
        if (j < d) {
          xk[j] = x;
          racc[q] += x + inv_mu * yv[q];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) W.gpart[warp * W.dstride + j] = racc[q];
    }
    __syncthreads();
    int bad = 0;
    for (int j = tid; j < d; j += kGenThreads) {  // admm.hpp:59
      float r = 0.0f;
#pragma unroll
      for (int i = 0; i < kGenWarps; ++i) r += W.gpart[i * W.dstride + j];
      const float zn = clamp_box(r / nf, box);
      W.z[j] = zn;
      bad |= !isfinite(zn);
    }
    __syncthreads();
    float rmax = 0.0f, oacc = 0.0f;
    bool rfin = true;
    for (int k = warp; k < n; k += kGenWarps) {  // admm.hpp:61-65
      const float* ak = a + static_cast<size_t>(k) * d;
      float* yk = ys + static_cast<size_t>(k) * d;
      const float* xk = xs + static_cast<size_t>(k) * d;
      float r2 = 0.0f, o2 = 0.0f;
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        if (j < d) {
          const float e = xk[j] - W.z[j];
          r2 = fmaf(e, e, r2);
          yk[j] += mu * e;
          if (want_obj) {
            const float t = W.z[j] - ak[j];
            o2 = fmaf(t, t, o2);
          }
        }
      }
      const float nr = sqrtf(warp_sum(r2));
      rfin &= isfinite(nr);
      rmax = fmaxf(rmax, nr);
      if (want_obj) oacc = fmaf(w[k], sqrtf(warp_sum(o2)), oacc);
    }
    if (lane == 0) {
      W.red[warp] = rfin ? rmax : __int_as_float(0x7fc00000);
      W.red[kGenWarps + warp] = oacc;
    }
    bad = __syncthreads_or(bad);
    float residual = 0.0f, obj = 0.0f;
    bool fin = true;
#pragma unroll
    for (int i = 0; i < kGenWarps; ++i) {
      fin &= isfinite(W.red[i]);
      residual = fmaxf(residual, W.red[i]);
      obj += W.red[kGenWarps + i];
    }
    __syncthreads();
    if (bad || !fin) {  // admm.hpp:67-68
      st.fail_iter = t;
      st.fail_kind = NLEM_FAIL_ADMM_ITERATE;
      return st;
    }
    if (want_obj) {  // admm.hpp:70-74
      if (!isfinite(obj)) {
        st.fail_iter = t;
        st.fail_kind = NLEM_FAIL_ADMM_OBJECTIVE;
        return st;
      }
      if (tid == 0) trace_obj[t - 1] = obj;
    }
    if (trace_res && tid == 0) trace_res[t - 1] = residual;
    on_iter(t, W.z);
    if (residual <= tol) {  // admm.hpp:77
      st.iterations = t;
      return st;
    }
  }
  return st;
}

// Block-wide p-form EM-ADMM on one problem.
//   a [n][d] points, w [n] weights, p state scratch of admm_state_floats(n, d) floats
//   W.z holds z0 on entry (visible to all threads), the minimizer on exit.
// on_iter(t, z) is called by every thread after sweep t (snapshots, nlem.cpp:92-128).
template <int JPL, class OnIter>
__device__ SolveStatus admm_solve_generic(const float* a, const float* w, float* p, int n, int d,
                                          GenWork& W, nlem_box box, float mu, int T, float tol,
                                          int res_mode, float* trace_obj, float* trace_res,
                                          OnIter on_iter, bool force_ref = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (force_ref || use_ref_form(n, d))
    return admm_solve_refform<JPL>(a, w, p + static_cast<size_t>(n) * d, p, n, d, W, box, mu, T,
                                   res_mode == RES_NONE ? -1.0f : tol, trace_obj, trace_res,
                                   on_iter);

  const float inv_mu = 1.0f / mu;
  const float nf = static_cast<float>(n);
  const bool want_obj = trace_obj != nullptr;
  const bool full = res_mode == RES_FULL;

  // static "all points equal a_0" for the exact-zero residual test
  int static_eq = 1;
  if (res_mode == RES_EXACT0) {
    int neq = 0;
    for (int e = tid; e < n * d; e += kGenThreads) neq |= (a[e] != a[e % d]);
    static_eq = !__syncthreads_or(neq);
  }

  SolveStatus st{T, -1, 0};
  // mode 0 = first (p = z0 - a), 1 = update, 2 = final (residual / objective only)
  auto pass = [&](int mode, bool& all1, bool& nrm_ok) {
    float gacc[JPL], zc[JPL], cc[JPL];
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      gacc[q] = 0.0f;
      zc[q] = j < d ? W.z[j] : 0.0f;
      cc[q] = j < d && mode == 1 ? 2.0f * W.z[j] - W.zprev[j] : 0.0f;
    }
    float rmax = 0.0f, oacc = 0.0f;
    all1 = true;
    nrm_ok = true;
    for (int k = warp; k < n; k += kGenWarps) {
      const float* ak = a + static_cast<size_t>(k) * d;
      float* pk = p + static_cast<size_t>(k) * d;
      float av[JPL], pv[JPL];
      float r2 = 0.0f, o2 = 0.0f;
      const float s_old = mode == 0 ? 0.0f : W.s[k];
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        av[q] = j < d ? ak[j] : 0.0f;
        if (mode == 0) {
          pv[q] = zc[q] - av[q];
        } else {
          pv[q] = j < d ? pk[j] : 0.0f;
          if (full) {
            const float e = fmaf(1.0f - s_old, pv[q], av[q] - zc[q]);
            r2 = fmaf(e, e, r2);
          }
          if (want_obj) {
            const float t = zc[q] - av[q];
            o2 = fmaf(t, t, o2);
          }
          if (mode == 1) pv[q] = fmaf(s_old, pv[q], cc[q] - av[q]);
        }
      }
      if (full) rmax = fmaxf(rmax, sqrtf(warp_sum(r2)));
      if (want_obj && mode != 0) oacc = fmaf(w[k], sqrtf(warp_sum(o2)), oacc);
      if (mode != 2) {
        float nr = 0.0f;
#pragma unroll
        for (int q = 0; q < JPL; ++q) nr = fmaf(pv[q], pv[q], nr);
        nr = warp_sum(nr);
        nrm_ok &= isfinite(nr);
        const float s = prox_scale(inv_mu * w[k], nr);
        all1 &= (s == 1.0f);
#pragma unroll
        for (int q = 0; q < JPL; ++q) {
          const int j = lane + 32 * q;
          gacc[q] = fmaf(s, pv[q], gacc[q]);
          if (j < d) pk[j] = pv[q];
        }
        if (lane == 0) W.s[k] = s;
      }
    }
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) W.gpart[warp * W.dstride + j] = gacc[q];
    }
    if (lane == 0) {
      W.red[warp] = rmax;
      W.red[kGenWarps + warp] = oacc;
    }
  };

  bool all1 = true, nrm_ok = true;
  pass(0, all1, nrm_ok);
  for (int t = 1; t <= T; ++t) {
    __syncthreads();
    // consensus z_t = P_C(z_{t-1} - g/n)   (admm.hpp:59)
    int bad = 0, neq = 0;
    for (int j = tid; j < d; j += kGenThreads) {
      float g = 0.0f;
#pragma unroll
      for (int i = 0; i < kGenWarps; ++i) g += W.gpart[i * W.dstride + j];
      const float zo = W.z[j];
      const float zn = clamp_box(zo - g / nf, box);
      W.zprev[j] = zo;
      W.z[j] = zn;
      bad |= !isfinite(zn);
      neq |= (zn != a[j]);
    }
    const int bad_z = __syncthreads_or(bad);
    const int bad_p = __syncthreads_or(!nrm_ok);
    const int any_neq = __syncthreads_or(neq);
    const int every1 = __syncthreads_and(all1);
    if (bad_z || bad_p) {
      // non-finite z_t (admm.hpp:67-68); a non-finite ||p_k|| produced by sweep t-1's
      // dual update is the multiplier blowing up, i.e. a non-finite residual of t-1
      st.fail_iter = (bad_z || t == 1) ? t : t - 1;
      st.fail_kind = NLEM_FAIL_ADMM_ITERATE;
      return st;
    }
    if (res_mode == RES_EXACT0 && static_eq && every1 && !any_neq) {
      on_iter(t, W.z);
      st.iterations = t;
      return st;
    }
    const bool last = t == T;
    float residual = 0.0f;
    if (full || want_obj || !last) {
      pass(last ? 2 : 1, all1, nrm_ok);
      __syncthreads();
      if (full) {
        for (int i = 0; i < kGenWarps; ++i) residual = fmaxf(residual, W.red[i]);
        // fmaxf drops NaN: re-check each partial
        bool fin = true;
        for (int i = 0; i < kGenWarps; ++i) fin &= isfinite(W.red[i]);
        if (!fin) residual = __int_as_float(0x7fc00000);
        if (!isfinite(residual)) {
          st.fail_iter = t;
          st.fail_kind = NLEM_FAIL_ADMM_ITERATE;
          return st;
        }
        if (trace_res && tid == 0) trace_res[t - 1] = residual;
      }
      if (want_obj) {
        float obj = 0.0f;
        for (int i = 0; i < kGenWarps; ++i) obj += W.red[kGenWarps + i];
        if (!isfinite(obj)) {
          st.fail_iter = t;
          st.fail_kind = NLEM_FAIL_ADMM_OBJECTIVE;
          return st;
        }
        if (tid == 0) trace_obj[t - 1] = obj;
      }
    }
    on_iter(t, W.z);
    if (full && residual <= tol) {
      st.iterations = t;
      return st;
    }
  }
  return st;
}

// Block-wide IRLS (proj/include/nlem/irls.hpp:21-68).  W.z holds x0 on entry and the
// minimizer on exit.  on_iter(t, x) receives the raw (unclamped) iterate.
template <int JPL, class OnIter>
__device__ SolveStatus irls_solve_generic(const float* a, const float* w, int n, int d, GenWork& W,
                                          float eps, int T, float tol, float* trace_obj,
                                          OnIter on_iter) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  SolveStatus st{T, -1, 0};
  // one pass at x = W.z: surrogate S(x) (costs.hpp:24-33), beta-weighted sums (irls.hpp:45-48)
  auto pass = [&]() {
    float xv[JPL], num[JPL];
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      xv[q] = j < d ? W.z[j] : 0.0f;
      num[q] = 0.0f;
    }
    float den = 0.0f, sur = 0.0f;
    for (int k = warp; k < n; k += kGenWarps) {
      const float* ak = a + static_cast<size_t>(k) * d;
      float av[JPL];
      float d2 = 0.0f;
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const int j = lane + 32 * q;
        av[q] = j < d ? ak[j] : 0.0f;
        const float t = xv[q] - av[q];
        d2 = fmaf(t, t, d2);
      }
      d2 = warp_sum(d2);
      const float root = sqrtf(d2 + eps);
      sur = fmaf(w[k], root, sur);
      const float beta = w[k] / root;
      den += beta;
#pragma unroll
      for (int q = 0; q < JPL; ++q) num[q] = fmaf(av[q], beta, num[q]);
    }
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const int j = lane + 32 * q;
      if (j < d) W.gpart[warp * W.dstride + j] = num[q];
    }
    if (lane == 0) {
      W.red[warp] = den;
      W.red[kGenWarps + warp] = sur;
    }
    __syncthreads();
    float S = 0.0f, D = 0.0f;
#pragma unroll
    for (int i = 0; i < kGenWarps; ++i) {
      D += W.red[i];
      S += W.red[kGenWarps + i];
    }
    return make_float2(S, D);
  };
  auto update = [&](float D) {  // x = num / den ; returns any non-finite
    int bad = 0;
    for (int j = tid; j < d; j += kGenThreads) {
      float g = 0.0f;
#pragma unroll
      for (int i = 0; i < kGenWarps; ++i) g += W.gpart[i * W.dstride + j];
      const float x = g / D;
      W.z[j] = x;
      bad |= !isfinite(x);
    }
    return __syncthreads_or(bad);
  };

  float2 SD = pass();
  float previous = SD.x;
  if (!isfinite(previous)) {
    st.fail_iter = 0;
    st.fail_kind = NLEM_FAIL_IRLS_OBJECTIVE;
    return st;
  }
  __syncthreads();
  if (update(SD.y)) {
    st.fail_iter = 1;
    st.fail_kind = NLEM_FAIL_IRLS_ITERATE;
    return st;
  }
  for (int t = 1; t <= T; ++t) {
    SD = pass();
    const float current = SD.x;
    if (!isfinite(current)) {
      st.fail_iter = t;
      st.fail_kind = NLEM_FAIL_IRLS_OBJECTIVE;
      return st;
    }
    if (trace_obj && tid == 0) trace_obj[t - 1] = current;
    on_iter(t, W.z);
    if (previous - current <= tol * fabsf(previous)) {
      st.iterations = t;
      return st;
    }
    previous = current;
    __syncthreads();
    if (t < T && update(SD.y)) {
      st.fail_iter = t + 1;
      st.fail_kind = NLEM_FAIL_IRLS_ITERATE;
      return st;
    }
  }
  return st;
}

}  // namespace nlemk
