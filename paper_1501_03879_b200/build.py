"""Build recipe for the in-tree sm_100a library (no torch extension, plain nvcc).

    python -m paper_1501_03879_b200.build        # -> paper_1501_03879_b200/_lib/libnlem_b200.so

The .so is git-ignored but travels to the GPU box with gpurun snapshots.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
SO = os.path.join(OUT_DIR, "libnlem_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["abi.cu", "kernels_generic.cu", "kernels_fast.cu", "kernels_nlem_tile.cu",
              "kernels_nlem_lr.cu", "kernels_nlem_lr_r12.cu", "kernels_batched_lr.cu",
              "kernels_aux.cu"]
CXX_SOURCES = ["synth.cpp", "multi_host.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
]


def sources():
    return [os.path.join(CSRC, s) for s in CU_SOURCES + CXX_SOURCES]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "nlem_b200.h"))
    if not os.path.exists(os.path.join(OUT_DIR, "nlem")):
        return True
    cli_deps = [os.path.join(HERE, "cli", "nlem_main.cpp"),
                os.path.join(os.path.dirname(HERE), "include", "nlem_b200.hpp"),
                os.path.join(os.path.dirname(HERE), "include", "nlem_b200_io.hpp")]
    return any(os.path.getmtime(p) > t for p in deps + cli_deps)


# experimental build variants (A/B and debug only): "_"-separated tokens -> defines
_VARIANT_TOKENS = {
    "prof": "-DNLEM_PHASE_PROFILE",  # tile kernel: clock64 phase stamps (nlem_debug_phase_times)
    "blrst": "-DNLEM_BLR_STAMPS",    # batched low-rank kernel: per-phase clock64 sums (printf)
    "cpt1": "-DNLEM_XW4_CPT=1",      # tile kernel: consensus threads per coordinate
    "cpt2": "-DNLEM_XW4_CPT=2",
    "cpt4": "-DNLEM_XW4_CPT=4",
    "cpt8": "-DNLEM_XW4_CPT=8",
    "lrst": "-DNLEM_LR_STAMPS",      # image low-rank kernel: per-phase clock64 sums (printf)
    "lrw4": "-DNLEM_LR_WARPS=4",     # image low-rank kernel: 4 pixel-warps per SM (unloaded phase latencies)
}


def variant_path(variant: str) -> str:
    return SO if not variant else SO.replace(".so", f"_{variant}.so")


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """variant="prof" etc.: debug / A-B builds into _lib/libnlem_b200_<variant>.so."""
    so = variant_path(variant)
    if not force and not variant and not _stale():
        return SO
    os.makedirs(OUT_DIR, exist_ok=True)
    toks = [t for t in variant.split("_") if t]
    extra = [_VARIANT_TOKENS[t] for t in toks if t in _VARIANT_TOKENS]
    # A/B against saved image-kernel versions (tools/dev/kernels_nlem_lr_*.cu): "lrr1" = round 1,
    # "lrnp2" = the rejected two-pixels-per-warp template (profiles/r2_np2_experiment.txt)
    swap = {}
    for tok, fname in (("lrr1", "kernels_nlem_lr_r1.cu"), ("lrnp2", "kernels_nlem_lr_np2_experiment.cu")):
        if tok in toks:
            swap[os.path.join(CSRC, "kernels_nlem_lr.cu")] = os.path.join(
                os.path.dirname(HERE), "tools", "dev", fname)
            extra += ["-I", CSRC]
    tag = f"_{variant}" if variant else ""
    jobs = []
    for src in sources():
        obj = os.path.join(OUT_DIR, os.path.basename(src) + tag + ".o")
        src = swap.get(src, src)
        if src.endswith(".cu"):
            cmd = [NVCC, *NVCC_FLAGS, *extra, "-c", src, "-o", obj]
        else:
            cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        jobs.append((cmd, obj))
    procs = [subprocess.Popen(cmd) for cmd, _ in jobs]  # one nvcc per translation unit
    failed = [cmd for (cmd, _), p in zip(jobs, procs) if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    objs = [obj for _, obj in jobs]
    tmp = so + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lpthread"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, so)
    for o in objs:
        os.remove(o)
    if not variant:
        build_cli(verbose)
    return so


CLI_SRC = os.path.join(HERE, "cli", "nlem_main.cpp")
CLI_BIN = os.path.join(OUT_DIR, "nlem")


def build_cli(verbose: bool = False) -> str:
    """The `nlem` command-line front end (host C++ over the C-ABI library, rpath $ORIGIN)."""
    inc = os.path.join(os.path.dirname(HERE), "include")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", inc, CLI_SRC, "-o", CLI_BIN + ".tmp",
           "-L", OUT_DIR, "-lnlem_b200", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(CLI_BIN + ".tmp", CLI_BIN)
    return CLI_BIN


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    if "--prof" in sys.argv:
        var = "prof"
    print(build(force="--force" in sys.argv, verbose=True, variant=var))
