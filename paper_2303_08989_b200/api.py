"""Python host mirror of the reference mpsgemm API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/
mpsgemm/*.hpp so the parity tests read like the reference's own tests.  Device
data lives in torch CUDA tensors (torch is plumbing here: allocation, streams,
H2D/D2H); every computation runs in libtcec_b200.so.

    h = Handle()                     # one handle per thread (owns stream + workspace)
    c, res = h.dispatch_cgemm(a, b, DispatchConfig(...))   # precsel.hpp:153-156
    c, ovf = h.cgemm(a, b, "FP16TCEC")                     # cgemm.hpp:17-18
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import DispatchConfig as _CConfig
from ._lib import DispatchResult, ExpStats, check

GEMM_MODES = {"FP32_REF": 0, "FP64_ORACLE": 1, "TF32TC": 2, "FP16TC": 3, "TF32TCEC": 4,
              "FP16TCEC": 5}
FORCED_MODES = {"FP32_REF": 0, "FP64_ORACLE": 1, "TF32TC": 2, "FP16TC": 3, "TF32TCEC": 4,
                "FP16TCEC": 5, "FP16TCEC_SCALED": 6}
KINDS = ["FP16TCEC", "FP16TCEC_SCALED", "TF32TCEC", "FP32_BASELINE"]
LEVELS = ["tf32_only", "fp16_scaled_ok", "fp16_ok"]


@dataclass
class SelectionPolicy:
    """precsel.hpp:60-65"""
    threshold_t: float = 0.0
    size_auto: int = 2048
    size_tf32: int = 512
    target_max_exponent: int = 14


def make_config(policy: SelectionPolicy | None = None, k_tile: int = 16,
                force: str | int | None = None) -> _CConfig:
    """DispatchConfig{policy, tiling, force} (precsel.hpp:140-144)."""
    p = policy or SelectionPolicy()
    f = -1 if force is None else (FORCED_MODES[force] if isinstance(force, str) else int(force))
    return _CConfig(float(p.threshold_t), int(p.size_auto), int(p.size_tf32),
                    int(p.target_max_exponent), int(k_tile), f, 0)


def _torch():
    import torch
    return torch


def _ptr(t) -> C.c_void_p:
    """Device pointer of a tensor the C-ABI may read as dense row-major memory.
    A strided view would be computed on the wrong layout, so it is rejected."""
    if not t.is_cuda:
        raise _lib.ShapeMismatch(1, "operand must be a CUDA tensor")
    if not t.is_contiguous():
        raise _lib.ShapeMismatch(1, "operand must be contiguous (call .contiguous())")
    return C.c_void_p(t.data_ptr())


class Handle:
    """tcec_handle: stream, workspace and device decision buffers of one thread."""

    def __init__(self, device: int = 0, stream=None):
        self.lib = _lib.load()
        self.device = device
        h = C.c_void_p()
        check(self.lib.tcec_create(device, C.byref(h)))
        self.h = h
        # networks bound to this handle: destroyed before the handle (a network
        # still alive when the handle closes would otherwise free its device
        # buffers through a dead handle)
        self._networks = weakref.WeakSet()
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "h", None):
            for net in list(getattr(self, "_networks", ())):
                net.close()
            self.lib.tcec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- control
    def set_stream(self, stream) -> None:
        ptr = stream if isinstance(stream, int) else (stream.cuda_stream if stream is not None else 0)
        check(self.lib.tcec_set_stream(self.h, C.c_void_p(ptr)))

    @property
    def stream_ptr(self) -> int:
        return self.lib.tcec_get_stream(self.h) or 0

    def synchronize(self) -> None:
        check(self.lib.tcec_synchronize(self.h))

    def _ordered_call(self, fn, *args):
        """Run one asynchronous device entry point on the handle stream, ordered
        after the work torch queued on its current stream (the operands) and
        before anything torch queues next (the results); then check its status."""
        torch = _torch()
        ext = self._ext_stream()
        cur = torch.cuda.current_stream(ext.device)
        if cur.cuda_stream != ext.cuda_stream:
            ext.wait_stream(cur)
        rc = fn(*args)
        if cur.cuda_stream != ext.cuda_stream:
            cur.wait_stream(ext)
        check(rc)

    def _ext_stream(self):
        """torch view of the handle stream (cached)."""
        torch = _torch()
        ptr = self.stream_ptr
        ext = getattr(self, "_ext", None)
        if ext is None or ext[0] != ptr:
            ext = (ptr, torch.cuda.ExternalStream(ptr, device=torch.device("cuda", self.device)))
            self._ext = ext
        return ext[1]

    @property
    def flush_kblocks(self) -> int:
        return self.lib.tcec_get_flush_kblocks(self.h)

    @flush_kblocks.setter
    def flush_kblocks(self, v: int) -> None:
        check(self.lib.tcec_set_flush_kblocks(self.h, int(v)))

    def set_executor(self, policy: int) -> None:
        """0 auto, 1 per-step permute+dispatch graph only, 2 fused small-step only,
        3 per-step graph preceded by the fused subtree launch (hybrid)."""
        check(self.lib.tcec_set_executor(self.h, int(policy)))

    GEMM_VARIANTS = {"auto": 0, "pair": 1, "single": 2, "wide": 3, "wide_persistent": 4, "wide_mc": 5,
                     "pair_persistent": 6}

    def set_operand_layout(self, layout) -> None:
        """tcec_set_operand_layout: "auto" (expand the smaller operand), "b" (B' =
        [[Br, Bi], [-Bi, Br]]) or "a" (A'' rows (Ar, -Ai) / (Ai, Ar))."""
        v = {"auto": 0, "b": 1, "a": 2}.get(layout, layout)
        check(self.lib.tcec_set_operand_layout(self.h, int(v)))

    def set_gemm_variant(self, variant) -> None:
        """tcgen05 kernel variant: "auto" (default), "pair" (cta_group::2,
        256x128 tile), "single" (128x128 tile), "wide" (cta_group::2, 256x256), "wide_persistent"
        (the same tile, persistent CTA pairs)."""
        v = self.GEMM_VARIANTS[variant] if isinstance(variant, str) else int(variant)
        check(self.lib.tcec_set_gemm_variant(self.h, v))

    def profile(self, on: bool = True) -> None:
        """Enable (and reset) per-stage CUDA-event tracing of dispatches."""
        check(self.lib.tcec_profile_enable(self.h, int(on)))

    def profile_read(self):
        """-> ({'stats': ms, 'prep': ms, 'gemm': ms}, n_dispatches)"""
        arr = (C.c_double * 3)()
        cnt = C.c_int64(0)
        check(self.lib.tcec_profile_read(self.h, arr, C.byref(cnt)))
        return {"stats": arr[0], "prep": arr[1], "gemm": arr[2]}, cnt.value

    def profile_read_batches(self):
        """-> (device ms summed over contraction batches from the end of their
        uploads to the start of their download, number of batches)"""
        ms, cnt = C.c_double(0.0), C.c_int64(0)
        check(self.lib.tcec_profile_read_batches(self.h, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def host_pipeline_stats(self):
        """-> (runs, reruns) of the pipelined host-buffer dispatch (reruns: the
        decision taken from the first operand parts differed from the exact one)."""
        runs, reruns = C.c_int64(0), C.c_int64(0)
        check(self.lib.tcec_host_pipeline_stats(self.h, C.byref(runs), C.byref(reruns)))
        return runs.value, reruns.value

    # ------------------------------------------------------ KernelTable level
    def _out_like(self, x):
        torch = _torch()
        if x.dtype != torch.float32:
            raise _lib.ShapeMismatch(1, f"buffer dtype must be float32, got {x.dtype}")
        if not x.is_cuda or x.device.index != self.device or not x.is_contiguous():
            raise _lib.ShapeMismatch(1, f"buffer must be a contiguous tensor on cuda:{self.device}")
        return torch.empty_like(x)

    def quantize_buf(self, x, fmt: int, rounding: int = 0):
        y = self._out_like(x)
        ovf = C.c_int(0)
        self._ordered_call(self.lib.tcec_quantize_buf, self.h, _ptr(x), _ptr(y), x.numel(), fmt, rounding,
                                         C.byref(ovf))
        return y, bool(ovf.value)

    def split_buf(self, x, fmt: int):
        hi, lo = self._out_like(x), self._out_like(x)
        ovf = C.c_int(0)
        self._ordered_call(self.lib.tcec_split_buf, self.h, _ptr(x), _ptr(hi), _ptr(lo), x.numel(), fmt,
                                      C.byref(ovf))
        return hi, lo, bool(ovf.value)

    def scale_buf(self, x, scale_exp: int):
        y = self._out_like(x)
        self._ordered_call(self.lib.tcec_scale_buf, self.h, _ptr(x), _ptr(y), x.numel(), int(scale_exp))
        return y

    def add_buf(self, a, b):
        y = self._out_like(a)
        self._out_like(b)
        if b.numel() != a.numel():
            raise _lib.ShapeMismatch(1, "add_buf: buffers differ in length")
        self._ordered_call(self.lib.tcec_add_buf, self.h, _ptr(a), _ptr(b), _ptr(y), a.numel())
        return y

    def sub_buf(self, a, b):
        y = self._out_like(a)
        self._out_like(b)
        if b.numel() != a.numel():
            raise _lib.ShapeMismatch(1, "sub_buf: buffers differ in length")
        self._ordered_call(self.lib.tcec_sub_buf, self.h, _ptr(a), _ptr(b), _ptr(y), a.numel())
        return y

    # ------------------------------------------------------------- precsel
    def exp_stats(self, m, target_max_exponent: int = 14) -> ExpStats:
        """exp_stats (precsel.hpp:68): both stages unconditionally."""
        out = ExpStats()
        self._check_c64(m)
        rows, cols = (m.shape if m.dim() == 2 else (1, m.numel()))
        self._ordered_call(self.lib.tcec_exp_stats, self.h, _ptr(m), rows, cols, target_max_exponent, 0, 0.0,
                                      C.byref(out))
        return out

    def exp_stats_staged(self, m, target_max_exponent: int, t: float) -> ExpStats:
        """exp_stats_staged (precsel.hpp:70)."""
        out = ExpStats()
        self._check_c64(m)
        rows, cols = (m.shape if m.dim() == 2 else (1, m.numel()))
        self._ordered_call(self.lib.tcec_exp_stats, self.h, _ptr(m), rows, cols, target_max_exponent, 1,
                                      float(t), C.byref(out))
        return out

    def scale_matrix_inplace(self, m, scale_exp: int) -> None:
        """scale_matrix_inplace (precsel.hpp:82): ScaleOverflow on nonfinite."""
        self._check_c64(m)
        x = m.view(_torch().float32)
        self._ordered_call(self.lib.tcec_scale_components, self.h, _ptr(x), x.numel(), int(scale_exp), 1)

    def scale_matrix(self, m, scale_exp: int):
        out = m.clone()
        self.scale_matrix_inplace(out, scale_exp)
        return out

    def descale_output_inplace(self, c, scale_exp_a: int, scale_exp_b: int) -> None:
        """descale_output_inplace (precsel.hpp:88): no overflow check."""
        self._check_c64(c)
        x = c.view(_torch().float32)
        self._ordered_call(self.lib.tcec_scale_components, self.h, _ptr(x), x.numel(),
                                             -(int(scale_exp_a) + int(scale_exp_b)), 0)

    # --------------------------------------------------------------- CGEMM
    def _check_c64(self, *ts):
        torch = _torch()
        for t in ts:
            if t.dtype != torch.complex64:
                raise _lib.ShapeMismatch(1, f"operand dtype must be complex64, got {t.dtype}")
            if not t.is_cuda or t.device.index != self.device:
                raise _lib.ShapeMismatch(1, f"operand must live on cuda:{self.device}")
            if not t.is_contiguous():
                raise _lib.ShapeMismatch(1, "operand must be contiguous (call .contiguous())")

    def _shapes(self, a, b):
        if a.dim() != 2 or b.dim() != 2:
            raise _lib.ShapeMismatch(1, "operands must be matrices")
        self._check_c64(a, b)
        m, k = a.shape
        k2, n = b.shape
        if k != k2:
            raise _lib.ShapeMismatch(1, "cgemm: inner dimensions differ")
        return m, n, k

    def cgemm(self, a, b, mode: str | int, k_tile: int = 16, out=None):
        """cgemm (cgemm.hpp:17-18); returns (C, overflow)."""
        m, n, k = self._shapes(a, b)
        c = out if out is not None else _torch().empty((m, n), dtype=_torch().complex64,
                                                       device=a.device)
        if out is not None:
            self._check_c64(c)
            if tuple(c.shape) != (m, n):
                raise _lib.ShapeMismatch(1, "output shape must be (m, n)")
        md = GEMM_MODES[mode] if isinstance(mode, str) else int(mode)
        ovf = C.c_int(0)
        self._ordered_call(self.lib.tcec_cgemm, self.h, _ptr(a), _ptr(b), _ptr(c), m, n, k, md, int(k_tile),
                                  C.byref(ovf))
        return c, bool(ovf.value)

    def cgemm_batched(self, pairs, mode, k_tile: int = 16):
        """cgemm_batched (cgemm.hpp:21-23): errors carry the batch index."""
        out = []
        for i, (a, b) in enumerate(pairs):
            try:
                out.append(self.cgemm(a, b, mode, k_tile)[0])
            except _lib.ShapeMismatch as e:
                raise _lib.ShapeMismatch(1, f"batch entry {i}: {e.msg}") from None
        return out

    def dispatch_cgemm(self, a, b, config: _CConfig | SelectionPolicy | None = None, out=None):
        """dispatch_cgemm (precsel.hpp:153-156); returns (C, DispatchResult)."""
        if config is None or isinstance(config, SelectionPolicy):
            config = make_config(config)
        m, n, k = self._shapes(a, b)
        c = out if out is not None else _torch().empty((m, n), dtype=_torch().complex64,
                                                       device=a.device)
        if out is not None:
            self._check_c64(c)
            if tuple(c.shape) != (m, n):
                raise _lib.ShapeMismatch(1, "output shape must be (m, n)")
        res = DispatchResult()
        self._ordered_call(self.lib.tcec_dispatch_cgemm, self.h, _ptr(a), _ptr(b), _ptr(c), m, n, k,
                                           C.byref(config), C.byref(res))
        return c, res

    def dispatch_cgemm_host(self, a: np.ndarray, b: np.ndarray, config=None, out=None):
        """The same with HOST numpy buffers (H2D / D2H inside the call)."""
        if config is None or isinstance(config, SelectionPolicy):
            config = make_config(config)
        a = np.ascontiguousarray(a, dtype=np.complex64)
        b = np.ascontiguousarray(b, dtype=np.complex64)
        m, k = a.shape
        n = b.shape[1]
        c = out if out is not None else np.empty((m, n), dtype=np.complex64)
        if b.shape[0] != k:
            raise _lib.ShapeMismatch(1, "dispatch_cgemm: inner dimensions differ")
        if c.dtype != np.complex64 or c.shape != (m, n) or not c.flags.c_contiguous:
            raise _lib.ShapeMismatch(1, "output must be a contiguous complex64 (m, n) array")
        res = DispatchResult()
        check(self.lib.tcec_dispatch_cgemm_host(self.h, a.ctypes.data_as(C.c_void_p),
                                                b.ctypes.data_as(C.c_void_p),
                                                c.ctypes.data_as(C.c_void_p), m, n, k,
                                                C.byref(config), C.byref(res)))
        return c, res

    # ------------------------------------------- operand preparation (test hook)
    def debug_prep(self, a, b, kind: str | int, scale_a: int = 0, scale_b: int = 0,
                   corrected: bool = True, xa: bool = False):
        """Run the hot path's prep_a / prep_b for a fixed decision and return the
        tensor-core operand planes (tcec_debug_prep_layout): A' hi/lo (m x kp) and
        B' hi/lo (2n x kp), binary16 for the FP16 kinds and f32 for TF32, plus the
        (format overflow, ScaleOverflow) flags.  xa=True: the A-expanded layout
        (A'' hi/lo 2m x kp, B'' hi/lo n x kp)."""
        torch = _torch()
        self._check_c64(a, b)
        kd = KINDS.index(kind) if isinstance(kind, str) else int(kind)
        m, k = a.shape
        k2, n = b.shape
        if k != k2:
            raise _lib.ShapeMismatch(1, "debug_prep: inner dimensions differ")
        kp = int(self.lib.tcec_prep_kp(k))
        dt = torch.float32 if kd == 2 else torch.float16
        ra, rb = (2 * m, n) if xa else (m, 2 * n)
        planes = [torch.zeros((r, kp), dtype=dt, device=a.device) for r in (ra, ra, rb, rb)]
        flags = (C.c_int * 2)()
        self._ordered_call(self.lib.tcec_debug_prep_layout, self.h, _ptr(a), _ptr(b), m, n, k, kd,
                           int(scale_a), int(scale_b), int(bool(corrected)), int(bool(xa)),
                           *[_ptr(t) for t in planes], flags)
        return (*planes, bool(flags[0]), bool(flags[1]))

    # ------------------------------------------------------------- permute
    def permute(self, t, axis_of):
        """permute (tensor.hpp:56-57): new axis a is old axis axis_of[a]."""
        r = t.dim()
        self._check_c64(t)
        if len(axis_of) != r:
            raise _lib.InvalidPermutation(4, "permutation has wrong length")
        out = _torch().empty(tuple(t.shape[a] for a in axis_of), dtype=t.dtype, device=t.device)
        dims = (C.c_int64 * max(r, 1))(*t.shape)
        ax = (C.c_int * max(r, 1))(*axis_of)
        self._ordered_call(self.lib.tcec_permute, self.h, _ptr(t), _ptr(out), r, dims, ax)
        return out


def matrix_tolerance(stats: ExpStats, t: float, target_max_exponent: int = 14) -> int:
    """matrix_tolerance (precsel.hpp:74): returns the ToleranceLevel index."""
    lib = _lib.load()
    lvl = C.c_int(0)
    check(lib.tcec_matrix_tolerance(C.byref(stats), float(t), target_max_exponent, C.byref(lvl)))
    return lvl.value


def select_mode(level_a: int, e_max_a, level_b: int, e_max_b, target_max_exponent: int = 14):
    """select_mode (precsel.hpp:76-77): returns (kind name, scale_a, scale_b)."""
    lib = _lib.load()
    k, sa, sb = C.c_int(0), C.c_int(0), C.c_int(0)
    check(lib.tcec_select_mode(level_a, e_max_a is not None, e_max_a or 0, level_b,
                               e_max_b is not None, e_max_b or 0, target_max_exponent,
                               C.byref(k), C.byref(sa), C.byref(sb)))
    return KINDS[k.value], sa.value, sb.value
