"""Benchmark inputs generated exactly as the reference generates them.

configs[1] (the CGEMM sweep, experiments.cpp:76-83): one Rng(seed + n), A then
B, two uniform_pm1f draws per complex element, row-major.  The generator is
the library's host restatement of rng.hpp (tcec_rng_*, std::mt19937_64 + the
reference's maps), so the device statistics and decision see the same operand
bits the reference's dispatch_cgemm sees.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check


class WorkloadRng:
    """Rng (rng.hpp:13-56) over the C-ABI: next_u64 / uniform_pm1f / gaussian streams."""

    def __init__(self, seed: int):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.tcec_rng_create(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.tcec_rng_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def next_u64(self) -> int:
        return int(self.lib.tcec_rng_next_u64(self.h))

    def fill_uniform_pm1f(self, out: np.ndarray) -> np.ndarray:
        """Fill a float32 (or complex64: re then im per element) array in place."""
        v = out.view(np.float32)
        assert v.flags.c_contiguous
        check(self.lib.tcec_rng_fill_uniform_pm1f(self.h, v.ctypes.data_as(C.c_void_p), v.size))
        return out

    def gaussian(self, n: int, stddev: float) -> np.ndarray:
        out = np.empty(n, np.float64)
        check(self.lib.tcec_rng_fill_gaussian(self.h, float(stddev), out.ctypes.data_as(C.c_void_p), n))
        return out


def sweep_operands(n: int, seed: int = 1, m: int | None = None, k: int | None = None,
                   pinned: bool = True):
    """A (m x k) then B (k x n) complex64 from Rng(seed + n): the configs[1]
    inputs of run_gemm_bench (experiments.cpp:80-83; square by default).
    Returned as host torch tensors (page-locked when a GPU is present)."""
    import torch
    m = n if m is None else m
    k = n if k is None else k
    pin = pinned and torch.cuda.is_available()
    a = torch.empty((m, k), dtype=torch.complex64, pin_memory=pin)
    b = torch.empty((k, n), dtype=torch.complex64, pin_memory=pin)
    r = WorkloadRng(seed + n)
    r.fill_uniform_pm1f(a.numpy())
    r.fill_uniform_pm1f(b.numpy())
    r.close()
    return a, b
