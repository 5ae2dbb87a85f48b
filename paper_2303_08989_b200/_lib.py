"""ctypes binding of the C-ABI in include/tcec_b200.h (libtcec_b200.so).

The library is loaded from the package directory (built in-tree by
paper_2303_08989_b200/build.py).  There is no fallback: if the library is
missing, or a compute call runs without an sm_100 GPU, an error is raised.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# TCEC_LIB_PATH: A/B of another build of the same C-ABI (development only)
LIB_PATH = os.environ.get("TCEC_LIB_PATH") or os.path.join(HERE, "libtcec_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tcec_b200.h")

STATUS = {
    0: "OK", 1: "ShapeMismatch", 2: "ZeroReference", 3: "ScaleOverflow",
    4: "InvalidPermutation", 5: "ExtentMismatch", 6: "InvalidPath",
    7: "DisconnectedNetwork", 8: "InvalidArgument", 9: "LogicError", 10: "CudaError",
    11: "TooManyQubits",
}


class TcecError(RuntimeError):
    """Base of the reference exception taxonomy (common.hpp:9-41)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class ShapeMismatch(TcecError, ValueError): pass
class ZeroReference(TcecError, ArithmeticError): pass
class ScaleOverflow(TcecError, OverflowError): pass
class InvalidPermutation(TcecError, ValueError): pass
class ExtentMismatch(TcecError, ValueError): pass
class InvalidPath(TcecError, ValueError): pass
class DisconnectedNetwork(TcecError, ValueError): pass
class InvalidArgument(TcecError, ValueError): pass
class LogicError(TcecError): pass
class CudaError(TcecError): pass
class TooManyQubits(TcecError, ValueError): pass


_EXC = {1: ShapeMismatch, 2: ZeroReference, 3: ScaleOverflow, 4: InvalidPermutation,
        5: ExtentMismatch, 6: InvalidPath, 7: DisconnectedNetwork, 8: InvalidArgument,
        9: LogicError, 10: CudaError, 11: TooManyQubits}


class ExpStats(C.Structure):
    """tcec_exp_stats_t == ExpStats (precsel.hpp:18-36)."""
    _fields_ = [("n1", C.c_uint64), ("n2", C.c_uint64), ("e_max_raw", C.c_int32),
                ("e_max_valid", C.c_int32), ("n_nonzero", C.c_uint64), ("n_total", C.c_uint64),
                ("stage2_evaluated_raw", C.c_int32), ("pad_", C.c_int32)]

    @property
    def e_max(self):
        return self.e_max_raw if self.e_max_valid else None

    @property
    def stage2_evaluated(self):
        return bool(self.stage2_evaluated_raw)

    def r1(self):
        return (self.n_nonzero - self.n1) / self.n_nonzero if self.n_nonzero else 0.0

    def r2(self):
        return (self.n_nonzero - self.n2) / self.n_nonzero if self.n_nonzero else 0.0

    def as_tuple(self):
        return (self.n1, self.n2, self.e_max, self.n_nonzero, self.n_total, self.stage2_evaluated)


class DispatchConfig(C.Structure):
    """tcec_dispatch_config_t == SelectionPolicy + TilingConfig + ForcedMode."""
    _fields_ = [("threshold_t", C.c_double), ("size_auto", C.c_int64), ("size_tf32", C.c_int64),
                ("target_max_exponent", C.c_int32), ("k_tile", C.c_int32), ("force", C.c_int32),
                ("pad_", C.c_int32)]


class DispatchResult(C.Structure):
    """tcec_dispatch_result_t == DispatchResult + DecisionRecord line."""
    _fields_ = [("kind", C.c_int32), ("scale_a", C.c_int32), ("scale_b", C.c_int32),
                ("overflow", C.c_int32), ("has_stats", C.c_int32), ("pad_", C.c_int32),
                ("stats_a", ExpStats), ("stats_b", ExpStats), ("line_raw", C.c_char * 160)]

    @property
    def line(self):
        return self.line_raw.decode()


_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tcec_[a-z0-9_]+)\s*\(", text)))


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the TCEC path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
    fp, ip = C.POINTER(C.c_float), C.POINTER(C.c_int)
    sig = {
        "tcec_last_error": ([], C.c_char_p),
        "tcec_version": ([], C.c_char_p),
        "tcec_create": ([i32, C.POINTER(vp)], i32),
        "tcec_destroy": ([vp], i32),
        "tcec_set_stream": ([vp, vp], i32),
        "tcec_get_stream": ([vp], vp),
        "tcec_synchronize": ([vp], i32),
        "tcec_set_flush_kblocks": ([vp, i32], i32),
        "tcec_get_flush_kblocks": ([vp], i32),
        "tcec_set_gemm_variant": ([vp, i32], i32),
        "tcec_set_operand_layout": ([vp, i32], i32),
        "tcec_get_operand_layout": ([vp], i32),
        "tcec_set_executor": ([vp, i32], i32),
        "tcec_profile_enable": ([vp, i32], i32),
        "tcec_profile_read": ([vp, C.POINTER(dbl), C.POINTER(i64)], i32),
        "tcec_host_pipeline_stats": ([vp, C.POINTER(i64), C.POINTER(i64)], i32),
        "tcec_profile_read_batches": ([vp, C.POINTER(dbl), C.POINTER(i64)], i32),
        "tcec_quantize_buf": ([vp, vp, vp, i64, i32, i32, ip], i32),
        "tcec_split_buf": ([vp, vp, vp, vp, i64, i32, ip], i32),
        "tcec_scale_buf": ([vp, vp, vp, i64, i32], i32),
        "tcec_add_buf": ([vp, vp, vp, vp, i64], i32),
        "tcec_sub_buf": ([vp, vp, vp, vp, i64], i32),
        "tcec_exp_stats": ([vp, vp, i64, i64, i32, i32, dbl, C.POINTER(ExpStats)], i32),
        "tcec_r1": ([C.POINTER(ExpStats)], dbl),
        "tcec_r2": ([C.POINTER(ExpStats)], dbl),
        "tcec_matrix_tolerance": ([C.POINTER(ExpStats), dbl, i32, ip], i32),
        "tcec_select_mode": ([i32] * 7 + [ip, ip, ip], i32),
        "tcec_scale_components": ([vp, vp, i64, i32, i32], i32),
        "tcec_cgemm": ([vp, vp, vp, vp, i64, i64, i64, i32, i32, ip], i32),
        "tcec_default_config": ([C.POINTER(DispatchConfig)], None),
        "tcec_dispatch_cgemm": ([vp, vp, vp, vp, i64, i64, i64, C.POINTER(DispatchConfig),
                                 C.POINTER(DispatchResult)], i32),
        "tcec_dispatch_cgemm_host": ([vp, vp, vp, vp, i64, i64, i64, C.POINTER(DispatchConfig),
                                      C.POINTER(DispatchResult)], i32),
        "tcec_permute": ([vp, vp, vp, i32, C.POINTER(i64), ip], i32),
        "tcec_network_create": ([vp, i32, ip, ip, C.POINTER(i64), C.POINTER(vp)], i32),
        "tcec_network_destroy": ([vp], i32),
        "tcec_network_set_node": ([vp, i32, vp], i32),
        "tcec_network_greedy_path": ([vp, ip], i32),
        "tcec_path_reconfigure": ([i32, ip, ip, C.POINTER(i64), ip, i32, i32, i32, i32, C.c_double,
                                   C.c_ulonglong, ip], i32),
        "tcec_contract_network": ([vp, ip, i32, C.POINTER(DispatchConfig), vp, i64, ip, ip,
                                   C.c_char_p, i64], i32),
        "tcec_contract_selector_batch": ([vp, ip, i32, C.POINTER(DispatchConfig), i32, ip, i32,
                                          C.POINTER(C.c_uint8), vp], i32),
        "tcec_contract_node_batch": ([vp, ip, i32, C.POINTER(DispatchConfig), i32, ip, i32, vp,
                                      vp], i32),
        "tcec_prep_kp": ([i64], i64),
        "tcec_network_step_results": ([vp, C.POINTER(DispatchResult), i32, ip], i32),
        "tcec_cgemm_oracle": ([vp, vp, vp, vp, i64, i64, i64], i32),
        "tcec_cgemm_c128": ([vp, vp, vp, vp, i64, i64, i64], i32),
        "tcec_permute_c128": ([vp, vp, vp, i32, C.POINTER(i64), ip], i32),
        "tcec_contract_network_oracle": ([vp, ip, i32, vp, i64, ip, ip], i32),
        "tcec_statevector_f64": ([vp, i32, i32, ip, ip, C.POINTER(C.c_double), vp], i32),
        "tcec_network_batch_run_info": ([vp, i32, ip, C.c_char_p, i64], i32),
        "tcec_rng_create": ([C.c_uint64, C.POINTER(vp)], i32),
        "tcec_rng_destroy": ([vp], i32),
        "tcec_rng_next_u64": ([vp], C.c_uint64),
        "tcec_rng_fill_uniform_pm1f": ([vp, vp, i64], i32),
        "tcec_rng_fill_gaussian": ([vp, dbl, vp, i64], i32),
        "tcec_debug_prep": ([vp, vp, vp, i64, i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, ip], i32),
        "tcec_debug_prep_layout": ([vp, vp, vp, i64, i64, i64, i32, i32, i32, i32, i32, vp, vp, vp, vp, ip],
                                   i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().tcec_last_error().decode()
        raise _EXC.get(rc, TcecError)(rc, msg)
