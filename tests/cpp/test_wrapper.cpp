// Reference-style KATs through the C++ host API (include/nlem_b200.hpp) -> C-ABI -> sm_100a.
// Mirrors proj/tests/unit/test_solvers.cpp:63-151 and test_denoise.cpp:165-179, 282-290.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <utility>

#include "nlem_b200.hpp"

static int failures = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);           \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

int main() {
  using namespace nlem;
  {  // single point from a distant start: one sweep, exact (test_solvers.cpp:64-82)
    PointSet ps{{0.0f, 0.0f}, {1.0f}, 2};
    AdmmConfig cfg;
    cfg.mu = 0.1f;
    cfg.max_iter = 2000;
    cfg.tol_primal = 1e-14f;
    cfg.z_init = {5.0f, 5.0f};
    SolverResult r = admm_euclidean_median(ps, BoxConstraint::unconstrained(), cfg);
    CHECK(r.iterations_run == 1);
    CHECK(r.minimizer[0] == 0.0f && r.minimizer[1] == 0.0f);
    CHECK(r.objective == 0.0f);
  }
  {  // documented recursion (test_solvers.cpp:122-151)
    PointSet ps{{0.0f, 1.0f}, {1.0f, 1.0f}, 1};
    AdmmConfig cfg;
    cfg.mu = 1.0f;
    cfg.max_iter = 3;
    cfg.record_trace = true;
    cfg.z_init = {0.25f};
    SolverResult r = admm_euclidean_median(ps, BoxConstraint::unconstrained(), cfg);
    CHECK(r.trace.size() == 3);
    CHECK(r.trace[0].objective == 1.0f && r.trace[0].primal_residual == 0.5f);
    CHECK(r.trace[1].objective == 1.0f && r.trace[1].primal_residual == 0.5f);
    CHECK(r.trace[2].primal_residual <= 1e-6f);
    CHECK(std::fabs(r.minimizer[0] - 0.5f) <= 1e-6f);
  }
  {  // IRLS single point (test_solvers.cpp:170-180)
    PointSet ps{{2.5f, 2.5f, 2.5f}, {1.0f}, 3};
    IrlsConfig cfg;
    cfg.max_iter = 1;
    SolverResult r = irls_euclidean_median(ps, cfg);
    CHECK(r.iterations_run == 1 && std::fabs(r.minimizer[1] - 2.5f) <= 1e-6f);
  }
  {  // validation -> std::invalid_argument (test_solvers.cpp:370-395)
    PointSet ps{{0.0f, 0.0f}, {1.0f}, 2};
    AdmmConfig bad;
    bad.mu = 0.0f;
    bool threw = false;
    try {
      admm_euclidean_median(ps, BoxConstraint::unconstrained(), bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  NlemParams params;  // small_params (test_denoise.cpp:74-84)
  params.search = 7;
  params.patch = 3;
  params.h = 30.0;
  params.sigma = 15.0;
  params.solver_iters = 4;
  {  // constant image is a fixed point (test_denoise.cpp:165-179)
    Image img(12, 10, 77.0f);
    Image out = nlem_denoise(img, params);
    bool all77 = true;
    for (int r = 0; r < 12; ++r)
      for (int c = 0; c < 10; ++c) all77 &= out(r, c) == 77.0f;
    CHECK(all77);
  }
  {  // snapshots forward-fill (test_denoise.cpp:282-290)
    Image img(8, 8, 50.0f);
    std::vector<Image> frames = nlem_denoise_snapshots(img, params);
    CHECK(frames.size() == 4);
    bool ok = true;
    for (const Image& f : frames)
      for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) ok &= f(r, c) == 50.0f;
    CHECK(ok);
  }
  {  // failure carries pixel coordinates (test_denoise.cpp:323-338)
    Image img(8, 8);
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) img(r, c) = ((r + c) % 2 == 0) ? 0.0f : 1e30f;
    NlemParams p = params;
    p.solver = DenoiseSolver::Irls;
    p.range = BoxConstraint::unconstrained();
    bool caught = false;
    try {
      nlem_denoise(img, p);
    } catch (const NumericFailure& e) {
      caught = std::string(e.what()).find("pixel (") != std::string::npos;
    }
    CHECK(caught);
  }
  {  // device pool (nlem_denoise_multi_host): 3 bands on device 0 == the single call, bitwise
    Image img(23, 17);
    for (int r = 0; r < 23; ++r)
      for (int c = 0; c < 17; ++c) img(r, c) = static_cast<float>((r * 37 + c * 11) % 256);
    Image one = nlem_denoise(img, params);
    Image three = nlem_denoise(img, params, std::vector<int32_t>{0, 0, 0});
    bool same = true;
    for (int r = 0; r < 23; ++r)
      for (int c = 0; c < 17; ++c) same &= one(r, c) == three(r, c);
    CHECK(same);
  }
  {  // solve_patch on a build_patch_stack stack (nlem.hpp:60-62, patch.cpp:90-114): the centre
     // coordinate of the solved patch is the pixel nlem_denoise writes (nlem.cpp:84)
    Image img(15, 13);
    for (int r = 0; r < 15; ++r)
      for (int c = 0; c < 13; ++c) img(r, c) = static_cast<float>((r * 53 + c * 29) % 200);
    NlemParams p = params;
    p.mu = 1.0;
    Image out = nlem_denoise(img, p);
    for (const auto& rc : {std::pair<int, int>{0, 0}, std::pair<int, int>{7, 6}, std::pair<int, int>{14, 12}}) {
      PatchStack st = build_patch_stack(img, rc.first, rc.second, p.search, p.patch, p.h);
      CHECK(st.d == 9 && st.weights[st.self_column] == 1.0f);
      PatchSolve s = solve_patch(st, p);
      std::vector<float> init = initial_patch(st, PatchInit::NoisyPatch);
      bool self = true;
      for (int j = 0; j < 9; ++j) self &= init[j] == st.patches[st.self_column * 9 + j] && s.init[j] == init[j];
      CHECK(self);
      CHECK(std::fabs(s.patch[4] - out(rc.first, rc.second)) <= 1e-2f);
    }
    PatchStack bad = build_patch_stack(img, 3, 3, 3, 3, 10.0);
    bad.self_column = 99;
    bool threw = false;
    try {
      solve_patch(bad, p);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("self column") != std::string::npos;
    }
    CHECK(threw);
  }
  CHECK(default_init_mode(60.5) == PatchInit::NlmPatch);
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
