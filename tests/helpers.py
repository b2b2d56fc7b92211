"""Shared input generators for the tests (seeded, numpy only)."""
from __future__ import annotations

import numpy as np


def solid_size(p: int) -> int:
    return p * (p + 1)


def random_solids(rng, n: int, p: int, dtype=np.float64, scale: float = 1.0) -> np.ndarray:
    """Normal coefficients with Im(C_n^0) = 0 (reference tests/test_helpers.hpp:16-27)."""
    x = rng.standard_normal((n, solid_size(p))) * scale
    for k in range(p):
        x[:, k * (k + 1) + 1] = 0.0
    return x.astype(dtype)


def random_shifts(rng, n: int, lo: float = 0.5, hi: float = 2.0, dtype=np.float64,
                  with_axes: bool = True) -> np.ndarray:
    """Uniform directions, |r| ~ U[lo, hi] (reference tests/test_helpers.hpp:29-39); the first
    rows are replaced by the axis-aligned shifts the reference tests single out
    (tests/test_pipeline.cpp:106-113)."""
    v = rng.standard_normal((n, 3))
    v *= rng.uniform(lo, hi, (n, 1)) / np.linalg.norm(v, axis=1, keepdims=True)
    if with_axes:
        axes = [[0, 0, 1.5], [0, 0, -1.5], [2.0, 0, 0], [-2.0, 0, 0], [0, 1.5, 0], [0, -1.5, 0]]
        for i, a in enumerate(axes[:n]):
            v[i] = a
    return v.astype(dtype)


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Numerically identical (signed zeros compare equal, NaNs in the same places)."""
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)


def glibc_hypot(x: float, y: float) -> float:
    """The algorithm csrc/device_math.cuh (hypot_ref) implements: glibc 2.39's
    __hypot for x86-64 (no-FMA kernel), restated with Python floats (IEEE double)."""
    import math
    if not (math.isfinite(x) and math.isfinite(y)):
        return math.inf if (math.isinf(x) or math.isinf(y)) else x + y
    x, y = abs(x), abs(y)
    ax, ay = (y, x) if x < y else (x, y)
    scale, large, tiny, eps = 2.0 ** -600, 2.0 ** 511, 2.0 ** -459, 2.0 ** -54

    def kernel(ax, ay):
        h = math.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            d = h - ay
            t1 = ax * (2.0 * d - ax)
            t2 = (d - 2.0 * (ax - ay)) * d
        else:
            d = h - ax
            t1 = 2.0 * d * (ax - 2.0 * ay)
            t2 = (4.0 * d - ay) * ay + d * d
        return h - (t1 + t2) / (2.0 * h)

    if ax > large:
        return ax + ay if ay <= ax * eps else kernel(ax * scale, ay * scale) / scale
    if ay < tiny:
        return ax + ay if ax >= ay / eps else kernel(ax / scale, ay / scale) * scale
    if ax >= ay / eps:
        return ax + ay
    return kernel(ax, ay)
