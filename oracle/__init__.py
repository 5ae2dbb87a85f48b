"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TCEC hot path.

ctypes bindings over
  * ``oracle/liboracle.so``          -- the plain-C restatement (tcec_oracle.c), and
  * ``oracle/_ref/libmpsgemm_ref.so`` -- the unmodified reference built in place
    (present only where ``/root/reference`` was available at build time).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package; the
product (``paper_2303_08989_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpsgemm_ref.so")
REF_SRC = "/root/reference/proj"

FMT_FP16, FMT_TF32 = 0, 1
RN, RZ = 0, 1
MODES = {"FP32_REF": 0, "FP64_ORACLE": 1, "TF32TC": 2, "FP16TC": 3, "TF32TCEC": 4, "FP16TCEC": 5}
FORCED = {"FP32_REF": 0, "FP64_ORACLE": 1, "TF32TC": 2, "FP16TC": 3, "TF32TCEC": 4,
          "FP16TCEC": 5, "FP16TCEC_SCALED": 6}
KINDS = ["FP16TCEC", "FP16TCEC_SCALED", "TF32TCEC", "FP32_BASELINE"]


class ExpStatsPod(C.Structure):
    _fields_ = [("n1", C.c_uint64), ("n2", C.c_uint64), ("e_max", C.c_int32),
                ("e_max_valid", C.c_int32), ("n_nonzero", C.c_uint64), ("n_total", C.c_uint64),
                ("stage2_evaluated", C.c_int32), ("pad_", C.c_int32)]

    def as_dict(self):
        return {"n1": self.n1, "n2": self.n2,
                "e_max": self.e_max if self.e_max_valid else None,
                "n_nonzero": self.n_nonzero, "n_total": self.n_total,
                "stage2_evaluated": bool(self.stage2_evaluated)}


class ConfigPod(C.Structure):
    _fields_ = [("threshold_t", C.c_double), ("size_auto", C.c_int64), ("size_tf32", C.c_int64),
                ("target_max_exponent", C.c_int32), ("k_tile", C.c_int32), ("force", C.c_int32),
                ("pad_", C.c_int32)]


class ResultPod(C.Structure):
    _fields_ = [("kind", C.c_int32), ("scale_a", C.c_int32), ("scale_b", C.c_int32),
                ("overflow", C.c_int32), ("has_stats", C.c_int32), ("pad_", C.c_int32),
                ("stats_a", ExpStatsPod), ("stats_b", ExpStatsPod), ("line", C.c_char * 160)]


class RngPod(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("have_spare", C.c_int),
                ("spare", C.c_double)]


def make_config(threshold_t=0.0, size_auto=2048, size_tf32=512, target=14, k_tile=16, force=None):
    """SelectionPolicy + TilingConfig + ForcedMode (precsel.hpp:60-65, :128-144)."""
    f = -1 if force is None else (FORCED[force] if isinstance(force, str) else int(force))
    return ConfigPod(float(threshold_t), int(size_auto), int(size_tf32), int(target), int(k_tile), f, 0)


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def build(with_ref: bool | None = None) -> None:
    """Compile liboracle.so (and the reference pin when /root/reference exists)."""
    targets = ["all"]
    if with_ref is None:
        with_ref = os.path.isdir(REF_SRC)
    if with_ref:
        targets += ["ref", "reftests"]  # reftests: the reference's own tests vs the drop-in
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib_cache: dict = {}


def _load(path):
    if path not in _lib_cache:
        _lib_cache[path] = C.CDLL(path)
    return _lib_cache[path]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


class _Backend:
    """Common numpy-facing API over either shared library (prefix orc_/ref_)."""

    def __init__(self, lib, prefix):
        self.lib = lib
        self.p = prefix
        self._sig()

    def f(self, name):
        return getattr(self.lib, self.p + name)

    def _sig(self):
        L, p = self.lib, self.p
        i64, f32, i32 = C.c_int64, C.c_float, C.c_int
        fp, dp = C.POINTER(C.c_float), C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        getattr(L, p + "quantize_buf").argtypes = [fp, fp, i64, i32, i32, ip]
        getattr(L, p + "split_buf").argtypes = [fp, fp, fp, i64, i32, ip]
        getattr(L, p + "scale_buf").argtypes = [fp, fp, i64, i32]
        getattr(L, p + "add_rz").argtypes = [f32, f32]
        getattr(L, p + "add_rz").restype = f32
        getattr(L, p + "exponent_of").argtypes = [f32, ip]
        getattr(L, p + "matrix_tolerance").argtypes = [C.POINTER(ExpStatsPod), C.c_double, i32]
        getattr(L, p + "select_mode").argtypes = [i32] * 7 + [ip, ip, ip]
        getattr(L, p + "cgemm").argtypes = [fp, fp, fp, i64, i64, i64, i32, i32, ip]
        getattr(L, p + "cgemm_oracle").argtypes = [fp, fp, dp, i64, i64, i64]
        getattr(L, p + "dispatch_cgemm").argtypes = [fp, fp, fp, i64, i64, i64,
                                                     C.POINTER(ConfigPod), C.POINTER(ResultPod)]
        getattr(L, p + "permute_c64").argtypes = [fp, fp, i32, C.POINTER(i64), ip]
        if p == "orc_":
            L.orc_dispatch_decision.argtypes = [fp, fp, i64, i64, i64, C.POINTER(ConfigPod),
                                                C.POINTER(ResultPod)]

    # --- lowprec / kernel table -------------------------------------------------
    def quantize_buf(self, x, fmt, rounding=RN):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        ovf = C.c_int(0)
        self.f("quantize_buf")(_fp(x), _fp(y), x.size, fmt, rounding, C.byref(ovf))
        return y, bool(ovf.value)

    def split_buf(self, x, fmt):
        x = np.ascontiguousarray(x, dtype=np.float32)
        hi, lo = np.empty_like(x), np.empty_like(x)
        ovf = C.c_int(0)
        self.f("split_buf")(_fp(x), _fp(hi), _fp(lo), x.size, fmt, C.byref(ovf))
        return hi, lo, bool(ovf.value)

    def scale_buf(self, x, s):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.empty_like(x)
        self.f("scale_buf")(_fp(x), _fp(y), x.size, int(s))
        return y

    def add_rz(self, a, b):
        return np.float32(self.f("add_rz")(float(a), float(b)))

    def exponent_of(self, x):
        e = C.c_int(0)
        ok = self.f("exponent_of")(float(np.float32(x)), C.byref(e))
        return e.value if ok else None

    # --- precsel ------------------------------------------------------------------
    def exp_stats(self, m, target=14):
        m = np.ascontiguousarray(m, dtype=np.complex64)
        out = ExpStatsPod()
        x = m.view(np.float32)
        if self.p == "orc_":
            self.lib.orc_exp_stats.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int,
                                               C.POINTER(ExpStatsPod)]
            self.lib.orc_exp_stats(_fp(x), 2 * m.size, target, C.byref(out))
        else:
            rows, cols = (m.shape if m.ndim == 2 else (1, m.size))
            self.lib.ref_exp_stats.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, C.c_int,
                                               C.POINTER(ExpStatsPod)]
            self.lib.ref_exp_stats(_fp(x), rows, cols, target, C.byref(out))
        return out

    def exp_stats_staged(self, m, target, t):
        m = np.ascontiguousarray(m, dtype=np.complex64)
        out = ExpStatsPod()
        x = m.view(np.float32)
        if self.p == "orc_":
            self.lib.orc_exp_stats_staged.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int,
                                                      C.c_double, C.POINTER(ExpStatsPod)]
            self.lib.orc_exp_stats_staged(_fp(x), 2 * m.size, target, float(t), C.byref(out))
        else:
            rows, cols = (m.shape if m.ndim == 2 else (1, m.size))
            self.lib.ref_exp_stats_staged.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64,
                                                      C.c_int, C.c_double, C.POINTER(ExpStatsPod)]
            self.lib.ref_exp_stats_staged(_fp(x), rows, cols, target, float(t), C.byref(out))
        return out

    def matrix_tolerance(self, stats, t, target=14):
        return self.f("matrix_tolerance")(C.byref(stats), float(t), target)

    def select_mode(self, la, ea, lb, eb, target=14):
        k, sa, sb = C.c_int(0), C.c_int(0), C.c_int(0)
        self.f("select_mode")(la, ea is not None, ea or 0, lb, eb is not None, eb or 0, target,
                              C.byref(k), C.byref(sa), C.byref(sb))
        return KINDS[k.value], sa.value, sb.value

    # --- gemm ---------------------------------------------------------------------
    def cgemm(self, a, b, mode, k_tile=16):
        a = np.ascontiguousarray(a, dtype=np.complex64)
        b = np.ascontiguousarray(b, dtype=np.complex64)
        m, k = a.shape
        k2, n = b.shape
        assert k == k2
        c = np.empty((m, n), dtype=np.complex64)
        ovf = C.c_int(0)
        md = MODES[mode] if isinstance(mode, str) else int(mode)
        rc = self.f("cgemm")(_fp(a.view(np.float32)), _fp(b.view(np.float32)),
                             _fp(c.view(np.float32)), m, n, k, md, k_tile, C.byref(ovf))
        if rc:
            raise RuntimeError(f"{self.p}cgemm failed rc={rc}")
        return c, bool(ovf.value)

    def cgemm_oracle(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.complex64)
        b = np.ascontiguousarray(b, dtype=np.complex64)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.complex128)
        self.f("cgemm_oracle")(_fp(a.view(np.float32)), _fp(b.view(np.float32)),
                               _dp(c.view(np.float64)), m, n, k)
        return c

    def dispatch_cgemm(self, a, b, cfg: ConfigPod):
        a = np.ascontiguousarray(a, dtype=np.complex64)
        b = np.ascontiguousarray(b, dtype=np.complex64)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.complex64)
        res = ResultPod()
        rc = self.f("dispatch_cgemm")(_fp(a.view(np.float32)), _fp(b.view(np.float32)),
                                      _fp(c.view(np.float32)), m, n, k, C.byref(cfg),
                                      C.byref(res))
        return rc, c, res

    def dispatch_decision(self, a, b, cfg: ConfigPod):
        """The selection half of dispatch_cgemm (oracle only): statistics,
        ComputeMode and the DecisionRecord line, no GEMM."""
        a = np.ascontiguousarray(a, dtype=np.complex64)
        b = np.ascontiguousarray(b, dtype=np.complex64)
        m, k = a.shape
        n = b.shape[1]
        res = ResultPod()
        rc = self.lib.orc_dispatch_decision(_fp(a.view(np.float32)), _fp(b.view(np.float32)), m, n, k,
                                            C.byref(cfg), C.byref(res))
        return rc, res

    def permute(self, t, axis_of):
        t = np.ascontiguousarray(t, dtype=np.complex64)
        r = t.ndim
        dims = (C.c_int64 * max(r, 1))(*t.shape)
        ax = (C.c_int * max(r, 1))(*axis_of)
        out = np.empty(tuple(t.shape[a] for a in axis_of), dtype=np.complex64)
        self.f("permute_c64")(_fp(t.view(np.float32)), _fp(out.view(np.float32)), r, dims, ax)
        return out


def oracle() -> _Backend:
    """The C restatement (always available once built)."""
    if not os.path.exists(ORACLE_SO):
        build(with_ref=False)
    return _Backend(_load(ORACLE_SO), "orc_")


def reference() -> _Backend | None:
    """The reference library itself, or None where it could not be built."""
    if not os.path.exists(REF_SO):
        return None
    return _Backend(_load(REF_SO), "ref_")


class Rng:
    """rng.hpp:13-56 via the C restatement (std::mt19937_64 + hand-rolled maps)."""

    def __init__(self, seed: int):
        self.lib = oracle().lib
        self.lib.orc_rng_next_u64.restype = C.c_uint64
        self.lib.orc_rng_next_below.restype = C.c_uint64
        self.lib.orc_rng_next_below.argtypes = [C.POINTER(RngPod), C.c_uint64]
        self.lib.orc_rng_uniform01.restype = C.c_double
        self.lib.orc_rng_uniform_pm1f.restype = C.c_float
        self.lib.orc_rng_gaussian.restype = C.c_double
        self.lib.orc_rng_gaussian.argtypes = [C.POINTER(RngPod), C.c_double]
        self.lib.orc_rng_seed.argtypes = [C.POINTER(RngPod), C.c_uint64]
        self.lib.orc_fill_uniform_c32.argtypes = [C.POINTER(RngPod), C.POINTER(C.c_float), C.c_int64]
        self.st = RngPod()
        self.lib.orc_rng_seed(C.byref(self.st), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF))

    def next_u64(self):
        return self.lib.orc_rng_next_u64(C.byref(self.st))

    def next_below(self, n):
        return self.lib.orc_rng_next_below(C.byref(self.st), n)

    def uniform01(self):
        return self.lib.orc_rng_uniform01(C.byref(self.st))

    def uniform_pm1f(self):
        return np.float32(self.lib.orc_rng_uniform_pm1f(C.byref(self.st)))

    def gaussian(self, sd):
        return self.lib.orc_rng_gaussian(C.byref(self.st), sd)

    def uniform_c32(self, rows, cols):
        """experiments.cpp:27-31 random_uniform_matrix."""
        m = np.empty((rows, cols), dtype=np.complex64)
        self.lib.orc_fill_uniform_c32(C.byref(self.st), _fp(m.view(np.float32)), m.size)
        return m
