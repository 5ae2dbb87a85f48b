"""Seeded input recipes shared by the golden generator and the tests.

All matrices come from the reference's Rng (rng.hpp:13-56) through the C
restatement (oracle.Rng), whose stream is pinned against the reference in
tests/golden/rng.json.
"""
from __future__ import annotations

import numpy as np

import oracle as O

SPECIALS = [0.0, -0.0, 2.0 ** -14, 2.0 ** -24, 2.0 ** -25, -(2.0 ** -30), 65504.0, 65520.0,
            2.0 ** -126, 2.0 ** -149, -1.1376953125 * 2.0 ** -130, 1.0 + 2.0 ** -11, 3.4e38, -3.4e38,
            0.99999994, -1.0000001, 70000.0, -65505.0, 1.0 + 2.0 ** -20, 2.0 ** -20, 1.5 * 2.0 ** -24,
            float("inf"), float("-inf"), float.fromhex("0x1.ffcp127"), float.fromhex("0x1.ffep127"), 2.0 ** 127]


def random_bits(seed: int, n: int) -> np.ndarray:
    """Random finite f32 values over the whole range (incl. subnormals)."""
    g = np.random.default_rng(seed)
    x = g.integers(0, 2 ** 32, n * 2, dtype=np.uint64).astype(np.uint32).view(np.float32)
    return np.ascontiguousarray(x[np.isfinite(x)][:n])


def matrix_recipe(name: str, rows: int, cols: int, seed: int) -> np.ndarray:
    r = O.Rng(seed)
    if name == "uniform":
        return r.uniform_c32(rows, cols)
    if name == "tiny20":
        return r.uniform_c32(rows, cols) * np.float32(2.0 ** -20)
    if name == "huge20":
        return r.uniform_c32(rows, cols) * np.float32(2.0 ** 20)
    if name == "subnormal":
        return r.uniform_c32(rows, cols) * np.float32(2.0 ** -130)
    if name == "zeros":
        return np.zeros((rows, cols), dtype=np.complex64)
    if name == "ones":
        return np.full((rows, cols), 1 + 1j, dtype=np.complex64)
    if name == "banded":
        # magnitudes in [0.1, 0.9] (test_precsel.cpp:263-276)
        v = np.empty(rows * cols * 2, dtype=np.float32)
        for i in range(v.size):
            v[i] = np.float32(0.1) + np.float32(0.8) * np.float32(r.uniform01())
        return v.view(np.complex64).reshape(rows, cols)
    if name == "mixed40":
        # 10% at 1.0, 90% at 2^-40 (test_precsel.cpp:95-103)
        m = np.empty(rows * cols, dtype=np.complex64)
        for i in range(m.size):
            mag = 1.0 if i % 10 == 0 else 2.0 ** -40
            m[i] = complex(mag, mag)
        return m.reshape(rows, cols)
    if name == "type3":
        # randtn Type 3 (network.cpp:402-434): N(0, 1e-2) * 1e-6 with 10-20 planted ones
        v = np.empty(rows * cols * 2, dtype=np.float32)
        for i in range(v.size):
            v[i] = np.float32(r.gaussian(1e-2)) * np.float32(1e-6)
        m = v.view(np.complex64).reshape(-1).copy()
        n_planted = 10 + r.next_below(11)
        for _ in range(min(n_planted, m.size)):
            m[r.next_below(m.size)] = 1.0 + 0.0j
        return m.reshape(rows, cols)
    if name == "sparse":
        m = r.uniform_c32(rows, cols).reshape(-1).copy()
        for i in range(m.size):
            if r.next_below(5) != 0:
                m[i] = 0
        return m.reshape(rows, cols)
    raise ValueError(name)
