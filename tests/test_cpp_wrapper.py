"""The C++ host API (include/nlem_b200.hpp) compiles against the C-ABI, and its
reference-style KATs pass on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp")


def _compile(out):
    from paper_1501_03879_b200 import _lib

    _lib.load()
    libdir = os.path.dirname(_lib.SO_PATH)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           "-L", libdir, "-lnlem_b200", f"-Wl,-rpath,{libdir}"]
    subprocess.run(cmd, check=True)


def test_cpp_wrapper_compiles(tmp_path):
    _compile(str(tmp_path / "t"))


@pytest.mark.gpu
def test_cpp_wrapper_kats(tmp_path):
    exe = str(tmp_path / "t")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
