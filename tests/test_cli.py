"""The `nlem` command-line front end (paper_1501_03879_b200/cli/nlem_main.cpp) and the host
file formats (include/nlem_b200_io.hpp), mirroring the reference's CLI contract
(proj/tools/nlem_main.cpp; proj/tests/unit/test_cli.cpp, test_pgm.cpp, test_point_set_io.cpp,
test_csv.cpp).  Usage / parse-error paths and the format KATs run on the CPU; every path that
solves something runs on the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    from paper_1501_03879_b200 import build as B

    B.build()  # no-op when fresh; builds the CLI next to the library
    if not os.path.exists(B.CLI_BIN):
        B.build_cli()
    return B.CLI_BIN


def run(cli, *args, timeout=600):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode() + np.clip(np.round(img), 0, 255).astype(np.uint8).tobytes())


def read_pgm(path):
    data = open(path, "rb").read()
    parts = data.split(b"\n", 3)
    assert parts[0] == b"P5"
    w, h = map(int, parts[1].split())
    return np.frombuffer(parts[3], np.uint8).reshape(h, w).astype(np.float64)


def read_csv(path):
    lines = open(path).read().splitlines()
    rows = [[float(x) if x else float("nan") for x in l.split(",")] for l in lines[1:]]
    return lines[0], rows


# ------------------------------------------------------------------------------------ CPU
def test_io_format_kats(tmp_path):
    from paper_1501_03879_b200 import _lib

    _lib.load()
    libdir = os.path.dirname(_lib.SO_PATH)
    exe = str(tmp_path / "test_io")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_io.cpp"), "-o", exe, "-L", libdir,
                    "-lnlem_b200", f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_usage_and_exit_codes(cli, tmp_path):
    """nlem_main.cpp:384-396: usage errors and malformed inputs exit 2 with "error:"."""
    assert run(cli, "--help")[0] == 0
    assert run(cli)[0] == 2
    assert run(cli, "frobnicate")[0] == 2
    code, out = run(cli, "median")
    assert code == 2 and "error:" in out
    code, out = run(cli, "median", tmp_path / "missing.txt")
    assert code == 2 and "cannot open point-set file" in out
    bad = tmp_path / "bad.txt"
    bad.write_text("2 2\n1 2 1\n3 x 1\n")
    code, out = run(cli, "median", bad)
    assert code == 2 and "byte offset" in out
    code, out = run(cli, "median", bad, "--solver", "gauss")
    assert code == 2
    code, out = run(cli, "median", bad, "--iters", "0")
    assert code == 2
    pgm = tmp_path / "bad.pgm"
    pgm.write_bytes(b"P5\n4 x\n255\n")
    code, out = run(cli, "denoise", pgm, "--out", tmp_path / "o.pgm")
    assert code == 2 and "malformed height" in out
    assert run(cli, "denoise", pgm)[0] == 2                       # --out required
    assert run(cli, "trace", pgm, "--trace", tmp_path / "t.csv")[0] == 2  # --pixel xor --psnr
    code, out = run(cli, "denoise", pgm, "--out", tmp_path / "o.pgm", "--patch", "4")
    assert code == 2 and "patch" in out                            # validate() before any I/O
    assert run(cli, "bench", pgm)[0] == 2                          # --sigma required


# ------------------------------------------------------------------------------------ GPU
def _points(tmp_path, pts, w):
    p = tmp_path / "pts.txt"
    n, d = pts.shape
    p.write_text(f"{n} {d}\n" + "".join(" ".join(f"{v:.17g}" for v in row) + f" {wk:.17g}\n"
                                        for row, wk in zip(pts, w)))
    return p


@pytest.mark.gpu
def test_median_subcommand(cli, tmp_path, oracle):
    # a single point is its own median (test_cli.cpp: exit 0, exact minimizer)
    code, out = run(cli, "median", _points(tmp_path, np.array([[5.0, 5.0]]), np.array([1.0])))
    assert code == 0, out
    rep = json.loads(out.splitlines()[-1])
    assert rep["minimizer"] == [5.0, 5.0] and rep["objective"] <= 1e-8 and rep["iterations"] >= 1
    # random set: ADMM (mu = 1, 200 sweeps) vs the FP64 oracle, with a trace CSV
    rng = np.random.default_rng(3)
    pts = rng.uniform(0.0, 1.0, (25, 3))
    w = rng.uniform(0.1, 1.0, 25)
    pf = _points(tmp_path, pts, w)
    tr = tmp_path / "trace.csv"
    code, out = run(cli, "median", pf, "--iters", 200, "--mu", 1.0, "--trace", tr)
    assert code == 0, out
    rep = json.loads(out.splitlines()[-1])
    ref = oracle.admm_batched(pts[None].astype(np.float32).astype(np.float64),
                              w[None].astype(np.float32).astype(np.float64), mu=1.0, max_iter=200)
    assert np.abs(np.array(rep["minimizer"]) - ref.minimizer[0]).max() <= 1e-4
    header, rows = read_csv(tr)
    assert header == "iter,objective,primal_residual" and len(rows) == rep["iterations"]
    assert all(np.isfinite(r[2]) for r in rows)
    # the box holds for both solvers
    for solver in ("admm", "irls"):
        code, out = run(cli, "median", pf, "--solver", solver, "--iters", 100, "--mu", 1.0,
                        "--range", "0.45:0.48")
        assert code == 0, out
        z = json.loads(out.splitlines()[-1])["minimizer"]
        assert all(0.45 - 1e-7 <= v <= 0.48 + 1e-7 for v in z)
    # float overflow in the sweep: NumericFailure -> exit 3
    code, out = run(cli, "median", _points(tmp_path, np.array([[3e38], [-3e38]]), np.array([1.0, 1.0])),
                    "--iters", 5, "--mu", 1.0)
    assert code == 3 and "error:" in out, out


@pytest.mark.gpu
def test_denoise_trace_bench_subcommands(cli, tmp_path):
    import paper_1501_03879_b200 as nb
    from paper_1501_03879_b200 import synth

    clean = np.round(synth.noisy_image(24, 24, 4, 3, 0.0)[0])
    src = tmp_path / "ramp.pgm"
    write_pgm(src, clean)
    out = tmp_path / "den.pgm"
    code, txt = run(cli, "denoise", src, "--sigma", 20, "--seed", 5, "--iters", 3, "--search", 11,
                    "--patch", 5, "--out", out)
    assert code == 0, txt
    assert "seed=5 psnr_noisy=" in txt and "psnr_denoised=" in txt
    den, noisy_pgm = read_pgm(out), read_pgm(tmp_path / "den_noisy.pgm")
    assert den.shape == (24, 24) and noisy_pgm.shape == (24, 24)
    # same result through the Python API on the same seeded noise
    noisy = synth.add_gaussian_noise(clean, 20.0, 5).astype(np.float32)
    p = nb.NlemParams(search=11, patch=5, h=200.0, sigma=20.0, solver="admm", solver_iters=3,
                      mu=1e-3, init_mode="noisy")
    ref = nb.nlem_denoise(noisy, p)
    assert np.abs(den - np.clip(np.round(ref), 0, 255)).max() <= 1.0
    psnr_d = float(txt.split("psnr_denoised=")[1].split()[0])
    mse = float(np.mean((clean - ref.astype(np.float64)) ** 2))
    assert abs(psnr_d - 10 * np.log10(255.0 ** 2 / mse)) <= 1e-3
    # repeated realizations and their mean line
    code, txt = run(cli, "denoise", src, "--sigma", 10, "--seed", 2, "--repeat", 3, "--iters", 2,
                    "--search", 7, "--patch", 3, "--out", out)
    assert code == 0 and all(f"seed={s} " in txt for s in (2, 3, 4)) and "mean psnr_noisy=" in txt
    # per-pixel objective trace (non-increasing for ADMM) and per-iteration PSNR table
    tr = tmp_path / "px.csv"
    code, txt = run(cli, "trace", src, "--sigma", 20, "--pixel", "5:7", "--iters", 6, "--mu", 1.0,
                    "--search", 11, "--patch", 5, "--trace", tr)
    assert code == 0, txt
    header, rows = read_csv(tr)
    assert header == "iter,objective,primal_residual" and len(rows) >= 2
    code, txt = run(cli, "trace", src, "--sigma", 20, "--psnr", "--iters", 4, "--search", 11,
                    "--patch", 5, "--trace", tr)
    assert code == 0, txt
    header, rows = read_csv(tr)
    assert header == "iter,psnr" and [r[0] for r in rows] == [1, 2, 3, 4]
    # bench table: images x sigmas x methods
    code, txt = run(cli, "bench", src, "--sigma", 10, 20, "--solver", "admm", "--solver", "nlm",
                    "--iters", 2, "--search", 7, "--patch", 3, "--repeat", 2)
    assert code == 0, txt
    lines = txt.strip().splitlines()
    assert lines[0] == "image,sigma,method,mean_psnr,std_psnr,R" and len(lines) == 1 + 4
    assert lines[1].startswith("ramp,10,admm,") and lines[1].endswith(",2")
