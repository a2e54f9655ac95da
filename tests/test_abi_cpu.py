"""CPU-side checks of the product library: it builds for sm_100a, loads, exports
every symbol include/nlem_b200.h declares, and its host-only pieces (parameter
validation, generators) behave like the reference.  No compute kernels run here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1501_03879_b200 import _lib as L
from paper_1501_03879_b200 import api, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_header_symbol():
    lib = L.load()
    header = open(os.path.join(ROOT, "include", "nlem_b200.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)  # declarations only
    declared = set(re.findall(r"\b(nlem_[a-z0-9_]+|nlm_denoise)\s*\(", header))
    declared -= {"nlem_status"}  # type name
    assert declared == set(L.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", L.SO_PATH], capture_output=True, text=True,
                         check=True).stdout
    for sym in declared:
        assert re.search(rf"\bT {sym}$", out, re.M), sym
        assert hasattr(lib, sym)
    assert b"sm_100a" in lib.nlem_version()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.SO_PATH],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_params_validation_messages():  # proj/src/nlm.cpp:17-29, test_denoise.cpp:88-123
    good = api.NlemParams(search=7, patch=3, h=30.0, sigma=15.0)
    api.validate(good)
    cases = [
        (dict(search=8), "search window must be odd and positive"),
        (dict(patch=9), "patch size must not exceed the search window"),
        (dict(patch=-3), "patch size must be odd and positive"),
        (dict(h=0.0), "similarity bandwidth h must be positive"),
        (dict(sigma=-1.0), "sigma must be nonnegative"),
        (dict(solver_iters=0), "solver_iters must be at least 1"),
        (dict(mu=0.0), "penalty mu must be positive"),
        (dict(epsilon=0.0), "epsilon must be positive"),
    ]
    for over, msg in cases:
        p = api.NlemParams(**{**good.__dict__, **over})
        with pytest.raises(api.InvalidArgument, match=msg):
            api.validate(p)
    with pytest.raises(api.InvalidArgument):
        api.BoxConstraint.interval(1.0, 0.0)


def test_default_init_mode():  # test_denoise.cpp:125-131
    for s, m in [(0.0, "noisy"), (30.0, "noisy"), (60.0, "noisy"), (60.5, "nlm"), (100.0, "nlm")]:
        assert api.default_init_mode(s) == m


def test_band_halo():
    assert api.band_halo(api.NlemParams(search=21, patch=7, h=1.0)) == 13


def test_noise_matches_oracle_bitwise(oracle):  # noise.hpp:15-40 restated twice
    clean = np.linspace(0, 255, 3000).reshape(50, 60)
    a = synth.add_gaussian_noise(clean, 20.0, 7)
    b = oracle.add_gaussian_noise(clean, 20.0, 7)
    assert (a == b).all()
    assert (synth.add_gaussian_noise(clean, 0.0, 3) == clean).all()


def test_image_generator_deterministic_and_in_range():
    c1, n1 = synth.noisy_image(128, 128, 12, 8, 20.0)
    c2, n2 = synth.noisy_image(128, 128, 12, 8, 20.0)
    assert (c1 == c2).all() and (n1 == n2).all()
    assert c1.min() >= 0 and c1.max() <= 255
    assert n1.max() > 255 or n1.min() < 0  # noise is not clipped
    resid = (n1 - c1).astype(np.float64)
    assert abs(resid.std() - 20.0) < 1.0
    # ramp visible where no shape was painted: first/last column differ by the ramp on average
    assert len(np.unique(c1)) > 20


def test_point_set_generator():
    p, w = synth.point_sets(4, 441, 49)
    p2, w2 = synth.point_sets(2, 441, 49, first=2)
    assert (p[2:] == p2).all() and (w[2:] == w2).all()
    assert (w > 0).all() and (w <= 1).all()
    inl = p[:, :397]
    assert 40 < inl.mean() < 210
    assert p[:, 397:].min() >= 0 and p[:, 397:].max() <= 255


def test_host_entry_rejects_bad_out_buffers():
    """A caller-supplied host `out` must be a writeable C-contiguous float32 array of the
    output shape (the C ABI writes rows*cols floats through its pointer) - checked before
    any device work."""
    p = api.NlemParams(search=7, patch=3, h=30.0, solver_iters=2)
    img = np.zeros((6, 5), np.float32)
    for bad in (np.zeros((6, 5), np.float64), np.zeros((5, 6), np.float32),
                np.zeros((6, 10), np.float32)[:, ::2], np.zeros(30, np.float32)):
        with pytest.raises(api.InvalidArgument, match="out must be"):
            api.nlem_denoise_host(img, p, out=bad)
    with pytest.raises(api.InvalidArgument, match="out must be"):
        api.nlem_denoise_rows_host(img, 0, 6, 5, 0, 3, p, out=np.zeros((6, 5), np.float32))
    with pytest.raises(api.InvalidArgument, match=r"\[in_rows\]\[cols\]"):
        api.nlem_denoise_rows_host(img[:, :4], 0, 6, 5, 0, 3, p)
