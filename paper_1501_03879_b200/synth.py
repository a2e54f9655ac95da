"""Seeded synthetic inputs of BASELINE.json's configs (host side, via the library's
C++ generators; exact recipe in csrc/synth.cpp and SURVEY.md §8d)."""
from __future__ import annotations

import numpy as np

from . import _lib as L

# BASELINE.json configs (image generators: rects, disks, sigma, size)
CONFIGS = {
    0: dict(rows=128, cols=128, rects=12, disks=8, sigma=20.0, patch=5, search=11, iters=20),
    2: dict(rows=512, cols=512, rects=40, disks=30, sigma=20.0, patch=7, search=21, iters=10),
    3: dict(rows=4096, cols=4096, rects=2000, disks=1500, sigma=30.0, patch=7, search=21, iters=10),
}


def noisy_image(rows, cols, rects, disks, sigma, image_seed=0, noise_seed=1):
    """(clean, noisy) float32 images."""
    clean = np.empty((rows, cols), np.float32)
    noisy = np.empty((rows, cols), np.float32)
    L.load().nlem_synth_noisy_image(rows, cols, rects, disks, float(sigma), image_seed, noise_seed,
                                    clean.ctypes.data, noisy.ctypes.data)
    return clean, noisy


def config_image(cfg: int, **over):
    c = dict(CONFIGS[cfg])
    c.update(over)
    return noisy_image(c["rows"], c["cols"], c["rects"], c["disks"], c["sigma"])


def point_sets(batch, n=441, d=49, seed_base=1000, first=0, threads=0, out=None):
    """Config-1 point sets: (points [B][n][d], weights [B][n]) float32."""
    pts = out[0] if out is not None else np.empty((batch, n, d), np.float32)
    w = out[1] if out is not None else np.empty((batch, n), np.float32)
    L.load().nlem_synth_point_sets(batch, n, d, seed_base, first, pts.ctypes.data, w.ctypes.data,
                                   threads)
    return pts, w


def add_gaussian_noise(clean, sigma, seed):
    """proj/src/noise.cpp:7-17 (float64 in/out, unclipped)."""
    clean = np.ascontiguousarray(clean, dtype=np.float64)
    out = np.empty_like(clean)
    L.load().nlem_add_gaussian_noise(clean.ctypes.data, clean.size, float(sigma), int(seed),
                                     out.ctypes.data)
    return out


def reference_h(sigma: float, d: int, mult: float = 10.0) -> float:
    """BASELINE weights exp(-D/(d h^2)) with h = mult*sigma == reference exp(-D/h_ref^2)
    with h_ref = h*sqrt(d)."""
    return float(mult * sigma * np.sqrt(d))
