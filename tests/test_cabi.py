"""The C-ABI boundary (include/tcec_b200.h / libtcec_b200.so) on a CPU-only box:
the library loads, exports every declared symbol, refuses to compute without
an sm_100 GPU (no CPU fallback), and its host-side logic (selection rule,
tolerance levels, log-line formatting, greedy path planning) matches the
reference."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_2303_08989_b200 import _lib
from paper_2303_08989_b200.api import matrix_tolerance, select_mode
from tests.golden.recipes import matrix_recipe


def test_library_exports_every_header_symbol():
    lib_path = _lib.LIB_PATH
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    lib = _lib.load()
    for s in syms:
        assert getattr(lib, s) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_tcgen05_and_tma_in_sass():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "UTCHMMA" in out or "UTCMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out                     # TMA loads
    assert "LDTM" in out                        # tcgen05.ld


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.tcec_create(0, C.byref(h))
    assert rc == 10  # TCEC_ERR_CUDA
    assert b"no CUDA device" in lib.tcec_last_error() or b"sm_100" in lib.tcec_last_error()
    from paper_2303_08989_b200 import CudaError, Handle
    with pytest.raises(CudaError):
        Handle(0)


def test_default_config_matches_reference_policy():
    lib = _lib.load()
    cfg = _lib.DispatchConfig()
    lib.tcec_default_config(C.byref(cfg))
    # SelectionPolicy{0, 2048, 512, 14} + TilingConfig{16} (precsel.hpp:60-65, gemm.hpp:28-30)
    assert (cfg.threshold_t, cfg.size_auto, cfg.size_tf32, cfg.target_max_exponent, cfg.k_tile,
            cfg.force) == (0.0, 2048, 512, 14, 16, -1)


def test_host_selection_logic_matches_reference_golden(golden):
    for c in golden("precsel.json")["select"]:
        assert select_mode(c["la"], c["ea"], c["lb"], c["eb"]) == (c["kind"], c["sa"], c["sb"])


def test_host_tolerance_logic_matches_oracle(orc, golden):
    for rec in golden("precsel.json")["stats"]:
        m = matrix_recipe(rec["recipe"], rec["rows"], rec["cols"], rec["seed"])
        for t, want in rec["level"].items():
            so = orc.exp_stats_staged(m, 14, float(t)).as_dict()
            st = _lib.ExpStats(so["n1"], so["n2"], so["e_max"] or 0, so["e_max"] is not None,
                               so["n_nonzero"], so["n_total"], int(so["stage2_evaluated"]), 0)
            if want < 0:
                with pytest.raises(_lib.LogicError):
                    matrix_tolerance(st, float(t))
            else:
                assert matrix_tolerance(st, float(t)) == want
            assert _lib.load().tcec_r1(C.byref(st)) == (
                (so["n_nonzero"] - so["n1"]) / so["n_nonzero"] if so["n_nonzero"] else 0.0)


def test_logic_error_when_stage2_skipped():
    # precsel.cpp:117-118
    st = _lib.ExpStats(0, 0, -20, 1, 10, 10, 0, 0)
    with pytest.raises(_lib.LogicError):
        matrix_tolerance(st, 0.0)


def test_greedy_path_planning_matches_reference_golden(golden):
    """tcec_network_greedy_path (C++ host planner, no device) == reference greedy_path."""
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.network import Network
    for rq in golden("rqc.json"):
        c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
        net = Network(None, circuit_to_network(c, [0] * c.n_qubits))
        assert [list(s) for s in net.greedy_path()] == rq["path"]
        net.close()


def test_greedy_path_random_networks_match_python_restatement():
    from oracle.network import greedy_path as py_greedy
    from paper_2303_08989_b200.circuits import NetworkSpec
    from paper_2303_08989_b200.network import Network
    g = np.random.default_rng(8)
    for it in range(30):
        n_nodes = int(g.integers(2, 9))
        spec = NetworkSpec()
        edges = []
        for e in range(int(g.integers(1, 14))):
            a, b = (int(v) for v in g.choice(n_nodes, 2, replace=False))
            edges.append((a, b, int(g.integers(2, 5))))
        for i in range(n_nodes):
            ls = [f"e{e}" for e, (a, b, _) in enumerate(edges) if i in (a, b)]
            ds = [d for (a, b, d) in edges if i in (a, b)]
            spec.labels.append(ls)
            spec.dims.append(ds)
            spec.data.append(np.zeros(int(np.prod(ds)) if ds else 1, np.complex64))
        net = Network(None, spec)
        assert net.greedy_path() == py_greedy(spec)
        net.close()


def test_network_validation_errors():
    from paper_2303_08989_b200.circuits import NetworkSpec
    from paper_2303_08989_b200.network import Network
    bad = NetworkSpec(labels=[["a"], ["a"], ["a"]], dims=[[2], [2], [2]],
                      data=[np.zeros(2, np.complex64)] * 3)
    net = Network(None, bad)
    with pytest.raises(_lib.ShapeMismatch):
        net.greedy_path()
    bad = NetworkSpec(labels=[["a"], ["a"]], dims=[[2], [3]],
                      data=[np.zeros(2, np.complex64), np.zeros(3, np.complex64)])
    net = Network(None, bad)
    with pytest.raises(_lib.ExtentMismatch):
        net.greedy_path()
