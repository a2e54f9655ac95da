"""Deterministic fixtures restated from the reference's test support
(proj/tests/support/synthetic.hpp) plus small helpers shared by the tests."""
import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def kats():
    with open(os.path.join(GOLDEN, "reference_kats.json")) as f:
        return json.load(f)


def house_like(n: int) -> np.ndarray:
    """proj/tests/support/synthetic.hpp:28-53 — piecewise-flat house scene."""
    img = np.empty((n, n))
    for r in range(n):
        for c in range(n):
            y = r / (n - 1)
            x = c / (n - 1)
            v = 185.0 - 20.0 * y
            if y > 0.95:
                v = 100.0
            roof = 0.18 <= y <= 0.45 and abs(x - 0.5) <= (y - 0.18) / 0.27 * 0.375
            chimney = 0.66 <= x <= 0.72 and 0.06 <= y <= 0.30 and not roof
            if chimney:
                v = 95.0
            if roof:
                v = 70.0
            if 0.45 < y <= 0.95 and 0.2 <= x <= 0.85:
                v = 120.0 if x > 0.62 else 155.0
                if 0.55 <= y <= 0.70 and ((0.28 <= x <= 0.40) or (0.66 <= x <= 0.78)):
                    v = 45.0
                if y >= 0.72 and 0.47 <= x <= 0.57:
                    v = 90.0
            img[r, c] = v
    return img


def texture_rich(n: int) -> np.ndarray:
    """proj/tests/support/synthetic.hpp:58-81."""
    img = np.empty((n, n))
    pi = math.pi
    for r in range(n):
        for c in range(n):
            y = r / (n - 1)
            x = c / (n - 1)
            if y < 0.5 and x < 0.5:
                v = 128.0 + 72.0 * math.sin(2.0 * pi * 9.0 * (x + y))
            elif y < 0.5:
                v = 128.0 + 72.0 * math.sin(2.0 * pi * 16.0 * x)
            elif x < 0.5:
                v = 60.0 + 150.0 * (x + (y - 0.5))
            else:
                a = (int(x * 16.0) + int(y * 16.0)) % 2 == 0
                v = 88.0 if a else 168.0
                v += 18.0 * math.sin(2.0 * pi * 20.0 * y)
            img[r, c] = v
    return img


def random_instance(rng: np.random.Generator, n: int, d: int, wlo=0.5, whi=1.5):
    """Same distribution as test_solvers.cpp:26-37 (coords U[0,1), weights U[0.5,1.5))."""
    pts = rng.uniform(0.0, 1.0, size=(n, d))
    w = rng.uniform(wlo, whi, size=n)
    return pts, w


def fold_index(i: int, n: int) -> int:
    """Independent step-by-step reflect oracle (test_patch.cpp:14-21)."""
    if n == 1:
        return 0
    while i < 0 or i >= n:
        if i < 0:
            i = -i
        if i >= n:
            i = 2 * (n - 1) - i
    return i
