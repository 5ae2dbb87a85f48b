"""B200-native (sm_100a) TCEC tensor-network contraction -- arXiv 2303.08989's
accelerator path rebuilt on tcgen05/TMA/TMEM behind the reference mpsgemm API.

The compute lives in libtcec_b200.so (include/tcec_b200.h); this package is the
Python host mirror used by the tests and the benchmark.
"""
from ._lib import (CudaError, DisconnectedNetwork, ExtentMismatch, InvalidArgument,  # noqa: F401
                   InvalidPath, InvalidPermutation, LogicError, ScaleOverflow, ShapeMismatch,
                   TcecError, TooManyQubits, ZeroReference, load)
from .api import (FORCED_MODES, GEMM_MODES, KINDS, Handle, SelectionPolicy,  # noqa: F401
                  make_config, matrix_tolerance, select_mode)
