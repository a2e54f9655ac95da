"""Writes tests/golden/reference_kats.json: the known-answer tests the reference's
own unit tests hold for the NLEM / EM-ADMM path, transcribed by hand (inputs,
expected outputs, tolerance) with the reference file:line each one comes from.

The reference keeps all KATs inline in its doctest files (no golden files exist,
SURVEY.md §4), so this script is the single place they are written down; both
the FP64 oracle (tests/test_oracle_kats.py) and the GPU path
(tests/test_gpu_parity.py) are checked against the JSON.

Run:  python tests/golden/make_reference_kats.py
"""
import json
import math
import os

T = "proj/tests/unit/"

KATS = {
    "mirror_index": {
        "source": T + "test_patch.cpp:44-50",
        "cases": [[-1, 5, 1], [-2, 5, 2], [5, 5, 3], [6, 5, 2]],  # (i, n, expected)
    },
    "corner_patch_2x2": {
        "source": T + "test_patch.cpp:52-59",
        "image": [[1, 2], [3, 4]], "row": 0, "col": 0, "k": 3,
        "expected": [4, 3, 4, 2, 1, 2, 4, 3, 4],
    },
    "weights_exp_minus_one": {
        "source": T + "test_patch.cpp:119-126",
        "patches": [[0, 0, 0, 0], [3, 0, 4, 0]], "center": 0, "h": 5.0,
        "expected": [1.0, math.exp(-1.0)], "rel_tol": 1e-15,
    },
    "corner_stack": {
        "source": T + "test_patch.cpp:150-168",
        "rows": 8, "cols": 8, "row": 0, "col": 0, "search": 5, "k": 3,
        "expected_n": 9, "expected_self_column": 0,
        "expected_neighbours": [[r, c] for r in range(3) for c in range(3)],
    },
    "interior_stack": {
        "source": T + "test_patch.cpp:170-179",
        "rows": 16, "cols": 16, "row": 8, "col": 8, "search": 7, "k": 3,
        "expected_n": 49, "expected_self_column": 24,
    },
    "prox_far_unit_pull": {
        "source": T + "test_prox.cpp:23-30",
        "v": [3.0, 4.0], "u": [0.0, 0.0], "lambda": 1.0, "expected": [2.4, 3.2], "rel_tol": 1e-15,
    },
    "prox_lands_on_u": {
        "source": T + "test_prox.cpp:31-35",
        "v": [3.0, 4.0], "u": [0.0, 0.0], "lambdas": [5.0, 7.25, "inf"], "expected": [0.0, 0.0],
    },
    "prox_zero_pull_identity": {
        "source": T + "test_prox.cpp:36-39",
        "v": [0.1 + 0.2, -7.5, 1e-300], "u": [1, 2, 3], "lambda": 0.0, "expected": [0.1 + 0.2, -7.5, 1e-300],
    },
    "prox_v_equals_u": {
        "source": T + "test_prox.cpp:40-43",
        "v": [1.0, 2.0], "u": [1.0, 2.0], "lambda": 0.5, "expected": [1.0, 2.0],
    },
    "ball_projection": {
        "source": T + "test_prox.cpp:126-143",
        "cases": [
            {"y": [0.3, 0.4], "radius": 0.5, "expected": [0.3, 0.4]},
            {"y": [3.0, 4.0], "radius": 1.0, "expected": [0.6, 0.8]},
            {"y": [3.0, 4.0], "radius": 0.0, "expected": [0.0, 0.0]},
        ],
    },
    "box_clamp": {
        "source": T + "test_prox.cpp:145-152",
        "x": [-5.0, 100.0, 300.0], "box": [0.0, 255.0], "expected": [0.0, 100.0, 255.0],
    },
    "em_cost_345": {
        "source": T + "test_costs.cpp:36-43",
        "points": [[0, 0], [3, 4]], "weights": [1, 1], "x": [0, 0], "expected": 5.0,
    },
    "surrogate_at_point": {
        "source": T + "test_costs.cpp:70-78",
        "points": [[0, 0]], "weights": [1], "x": [0, 0], "eps": 1.0, "expected": 1.0,
    },
    "admm_single_point_distant_start": {
        "source": T + "test_solvers.cpp:64-82",
        "points": [[0.0, 0.0]], "weights": [1.0], "mu": 0.1, "max_iter": 2000,
        "tol_primal": 1e-14, "z_init": [5.0, 5.0],
        "expected_iterations": 1, "expected_minimizer": [0.0, 0.0], "expected_objective": 0.0,
    },
    "admm_single_point_undersized_radius": {
        "source": T + "test_solvers.cpp:83-99",
        "points": [[0.0, 0.0]], "weights": [1.0], "mu": 0.5, "max_iter": 2000,
        "tol_primal": 0.0, "z_init": [3.0, 4.0],
        "expected_iterations": 1, "expected_objective": 3.0,
    },
    "admm_single_point_default_start": {
        "source": T + "test_solvers.cpp:100-110",
        "points": [[-3.0, 8.0]], "weights": [1.0], "mu": 1e-3, "max_iter": 100,
        "tol_primal": 0.0, "z_init": None,
        "expected_minimizer": [-3.0, 8.0], "expected_objective": 0.0,
    },
    "admm_equilateral_triangle": {
        "source": T + "test_solvers.cpp:111-119 (admm_converged :43-49: mu = 2*mean(w))",
        "points": [[0.0, 0.0], [1.0, 0.0], [0.5, math.sqrt(3.0) / 2.0]], "weights": [1, 1, 1],
        "mu": 2.0, "max_iter": 100000, "tol_primal": 0.0,
        "expected_minimizer": [0.5, math.sqrt(3.0) / 6.0], "rel_tol": 1e-6,
        "expected_objective": math.sqrt(3.0), "objective_rel_tol": 1e-9,
    },
    "admm_recursion": {
        "source": T + "test_solvers.cpp:122-151",
        "points": [[0.0], [1.0]], "weights": [1.0, 1.0], "mu": 1.0, "max_iter": 3,
        "z_init": [0.25],
        "expected_trace_objective": [1.0, 1.0], "expected_trace_residual": [0.5, 0.5],
        "third_residual_max": 1e-12, "expected_minimizer": [0.5], "expected_objective": 1.0,
    },
    "irls_single_point": {
        "source": T + "test_solvers.cpp:170-180",
        "points": [[2.5, 2.5, 2.5]], "weights": [1.0], "epsilon": 1e-6, "max_iter": 1,
        "expected_minimizer": [2.5, 2.5, 2.5], "expected_iterations": 1,
    },
    "irls_equilateral_corner_start": {
        "source": T + "test_solvers.cpp:181-191",
        "points": [[0.0, 0.0], [1.0, 0.0], [0.5, math.sqrt(3.0) / 2.0]], "weights": [1, 1, 1],
        "epsilon": 1e-6, "max_iter": 2000, "x_init": [0.0, 0.0],
        "expected_minimizer": [0.5, math.sqrt(3.0) / 6.0], "rel_tol": 1e-5,
    },
    "admm_overflow": {
        "source": T + "test_solvers.cpp:342-362",
        "points": [[0.0, 0.0], [10.0, 0.0]], "weights": [1e308, 1e308], "mu": 1.0,
        "max_iter": 5, "record_trace": True, "expect": "NumericFailure objective",
    },
    "nlem_constant_image": {
        "source": T + "test_denoise.cpp:165-179 (small_params :74-84)",
        "rows": 12, "cols": 10, "value": 77.0,
        "params": {"search": 7, "patch": 3, "h": 30.0, "sigma": 15.0, "solver_iters": 4,
                   "mu": 1e-3, "epsilon": 1e-6, "init_mode": "noisy"},
        "expected_admm": 77.0, "expected_nlm": 77.0, "irls_abs_tol": 1e-9,
    },
    "nlem_snapshot_forward_fill": {
        "source": T + "test_denoise.cpp:282-290",
        "rows": 8, "cols": 8, "value": 50.0, "solver_iters": 4, "expected": 50.0,
    },
    "default_init_mode": {
        "source": T + "test_denoise.cpp:125-131",
        "cases": [[0.0, "noisy"], [30.0, "noisy"], [60.0, "noisy"], [60.5, "nlm"], [100.0, "nlm"]],
    },
    "noise_psnr_closed_form": {
        "source": T + "test_noise.cpp:56-63",
        "sigma": 40.0, "seed": 2026, "expected_psnr": 20 * math.log10(255 / 40.0), "rel_tol": 0.005,
    },
}


def main():
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_kats.json")

    def enc(o):
        if isinstance(o, float) and math.isinf(o):
            return "inf"
        return o

    with open(out, "w") as f:
        json.dump(KATS, f, indent=1, default=enc)
        f.write("\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
