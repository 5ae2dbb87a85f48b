"""The CPU oracle (oracle/tcec_oracle.c) against the reference's golden vectors
(tests/golden/*, produced by tests/golden/make_golden.py from the reference)
and the reference's own known-answer tests.  Runs everywhere (no GPU)."""
import hashlib

import numpy as np
import pytest

import oracle as O
from tests.conftest import bits
from tests.golden.recipes import SPECIALS, matrix_recipe


# ---------------------------------------------------------------- lowprec KATs
# reference tests/test_lowprec.cpp:40-204
def test_exponent_of_kats(orc):
    assert orc.exponent_of(1.0) == 0
    assert orc.exponent_of(0.75) == -1
    assert orc.exponent_of(0.0) is None and orc.exponent_of(-0.0) is None
    assert orc.exponent_of(2.0) == 1
    assert orc.exponent_of(2.0 ** -126) == -126
    assert orc.exponent_of(2.0 ** -149) == -149
    assert orc.exponent_of(1.5 * 2.0 ** -140) == -140
    assert orc.exponent_of(-3.0) == 1


def _q(orc, x, fmt, rd=O.RN):
    y, ovf = orc.quantize_buf(np.array([x], np.float32), fmt, rd)
    return y[0], ovf


def test_quantize_kats(orc):
    f16, tf32 = O.FMT_FP16, O.FMT_TF32
    assert _q(orc, 1.0, f16)[0] == 1.0
    assert _q(orc, 1.0 + 2.0 ** -12, f16)[0] == 1.0
    assert _q(orc, 1.0 + 2.0 ** -12, tf32)[0] == 1.0
    assert _q(orc, 2.0 ** -30, f16)[0] == 0.0
    assert _q(orc, 2.0 ** -20, f16)[0] == np.float32(2.0 ** -20)
    assert _q(orc, 1.015625 * 2.0 ** -20, f16)[0] == np.float32(2.0 ** -20)
    assert _q(orc, 1.0 + 2.0 ** -11, f16)[0] == 1.0  # tie to even
    assert _q(orc, 1.0 + 1.5 * 2.0 ** -11, f16)[0] == np.float32(1.0 + 2.0 ** -10)
    assert _q(orc, 1.0 + 1.9375 * 2.0 ** -11, f16, O.RZ)[0] == 1.0
    assert np.signbit(_q(orc, -0.0, f16)[0])
    # saturation (test_lowprec.cpp:81-105)
    assert _q(orc, 70000.0, f16) == (65504.0, True)
    assert _q(orc, -65504.0, f16) == (-65504.0, False)
    assert _q(orc, 65505.0, f16, O.RZ) == (65504.0, True)
    r, ovf = _q(orc, np.finfo(np.float32).max, tf32)
    assert ovf and r == np.float32(float.fromhex("0x1.ffcp127"))


def test_split_kats(orc):
    hi, lo, _ = orc.split_buf(np.array([1.0, 1.0 + 2.0 ** -20], np.float32), O.FMT_FP16)
    assert hi[0] == 1.0 and lo[0] == 0.0
    assert hi[1] == 1.0 and lo[1] == np.float32(2.0 ** -9)


def test_add_rz_kats(orc):
    assert orc.add_rz(1.0, 1.5 * 2.0 ** -24) == 1.0
    assert orc.add_rz(-1.0, -1.5 * 2.0 ** -24) == -1.0
    assert orc.add_rz(0.5, 0.25) == 0.75
    assert orc.add_rz(1.0, -1.0) == 0.0


def test_lowprec_vectors_match_reference_golden(orc, golden):
    g = golden("lowprec.npz")
    x = g["x"].view(np.float32)
    for fmt in (0, 1):
        for rd in (0, 1):
            q, ovf = orc.quantize_buf(x, fmt, rd)
            assert np.array_equal(bits(q), g[f"q{fmt}{rd}"]), (fmt, rd)
            assert ovf == bool(g[f"q{fmt}{rd}_ovf"][0])
            each = [orc.quantize_buf(np.array([v], np.float32), fmt, rd)[1] for v in SPECIALS]
            assert each == list(g[f"q{fmt}{rd}_ovf_each"])
        hi, lo, ovf = orc.split_buf(x, fmt)
        assert np.array_equal(bits(hi), g[f"hi{fmt}"]) and np.array_equal(bits(lo), g[f"lo{fmt}"])
        assert ovf == bool(g[f"s{fmt}_ovf"][0])
    for s in (0, 1, -7, 34, -163, 163, 1100):
        assert np.array_equal(bits(orc.scale_buf(x, s)), g[f"scale{s}"]), s


# ------------------------------------------------------------------ rng pin
def test_rng_matches_reference_stream(golden):
    g = golden("rng.json")
    for seed in (1, 42, 1 ^ 0xC2B2AE3D27D4EB4F):
        r = O.Rng(seed)
        assert [float(r.next_u64() >> 11) for _ in range(64)] == g[f"{seed}:0"]
        r = O.Rng(seed)
        assert [float(r.next_below(1000003)) for _ in range(64)] == g[f"{seed}:1"]
        r = O.Rng(seed)
        assert [r.gaussian(1e-2) for _ in range(64)] == g[f"{seed}:2"]
        r = O.Rng(seed)
        assert [r.uniform01() for _ in range(64)] == g[f"{seed}:3"]
        m = O.Rng(seed).uniform_c32(4, 5)
        assert bits(m.view(np.float32)).tolist() == g[f"{seed}:uniform_c32"]


def test_python_rng_matches_oracle_rng():
    from paper_2303_08989_b200.circuits import Rng as PyRng
    for seed in (1, 5, 2 ** 63 + 7):
        a, b = O.Rng(seed), PyRng(seed)
        assert [a.next_u64() for _ in range(700)] == [b.next_u64() for _ in range(700)]
        assert [a.next_below(3) for _ in range(50)] == [b.next_below(3) for _ in range(50)]
        assert [a.gaussian(1e-2) for _ in range(20)] == [b.gaussian(1e-2) for _ in range(20)]


# ----------------------------------------------------------- stats / select
def test_stats_and_levels_match_reference_golden(orc, golden):
    for rec in golden("precsel.json")["stats"]:
        m = matrix_recipe(rec["recipe"], rec["rows"], rec["cols"], rec["seed"])
        assert orc.exp_stats(m).as_dict() == rec["full"], rec["recipe"]
        for t, want in rec["staged"].items():
            st = orc.exp_stats_staged(m, 14, float(t))
            assert st.as_dict() == want, (rec["recipe"], t)
            assert orc.matrix_tolerance(st, float(t), 14) == rec["level"][t]


def test_select_mode_matches_reference_golden(orc, golden):
    for c in golden("precsel.json")["select"]:
        assert orc.select_mode(c["la"], c["ea"], c["lb"], c["eb"]) == (c["kind"], c["sa"], c["sb"])


def test_stats_kats(orc):
    # test_precsel.cpp:30-86
    ones = np.full((4, 4), 1 + 1j, np.complex64)
    s = orc.exp_stats(ones).as_dict()
    assert (s["n_total"], s["n_nonzero"], s["n1"], s["e_max"]) == (32, 32, 32, 0)
    tiny = np.full((4, 4), (1 + 1j) * 2.0 ** -20, np.complex64)
    s = orc.exp_stats(tiny).as_dict()
    assert s["n1"] == 0 and s["e_max"] == -20 and s["n2"] == s["n_nonzero"]
    m = np.array([[1.0, 2.0 ** -40]], np.complex64)
    s = orc.exp_stats(m).as_dict()
    assert (s["e_max"], s["n_nonzero"], s["n1"], s["n2"]) == (0, 2, 1, 1)
    s = orc.exp_stats(np.zeros((3, 3), np.complex64)).as_dict()
    assert s["e_max"] is None and s["n_nonzero"] == 0
    skipped = orc.exp_stats_staged(np.full((4, 4), 0.5, np.complex64), 14, 0.0).as_dict()
    assert not skipped["stage2_evaluated"] and skipped["n2"] == skipped["n1"]


def test_log_line_kat(orc):
    # test_precsel.cpp:324-349 through the oracle's dispatch formatting
    cfg = O.make_config(force="FP32_REF")
    a = np.ones((64, 64), np.complex64)
    rc, _, res = orc.dispatch_cgemm(a, a, O.make_config())
    assert rc == 0 and res.line.decode() == "64,64,64,FP32_BASELINE,0,0,-,-,-,-,-,-"
    rc, _, res = orc.dispatch_cgemm(a, a, cfg)
    assert res.line.decode() == "64,64,64,FP32_REF,0,0,-,-,-,-,-,-"


# -------------------------------------------------------------------- cgemm
def test_cgemm_all_modes_match_reference_golden(orc, golden):
    g = golden("cgemm.npz")
    for (m, n, k) in [(1, 1, 1), (3, 5, 7), (8, 32, 16), (13, 37, 65), (16, 48, 33), (64, 64, 64),
                      (100, 1, 50), (1, 200, 3)]:
        a = matrix_recipe("uniform", m, k, 1000 + m)
        b = matrix_recipe("uniform", k, n, 2000 + n)
        for mode in O.MODES:
            c, _ = orc.cgemm(a, b, mode)
            assert np.array_equal(bits(c.view(np.float32)), g[f"{m}x{n}x{k}:{mode}"]), (m, n, k, mode)
        assert np.array_equal(orc.cgemm_oracle(a, b).view(np.float64), g[f"{m}x{n}x{k}:oracle"])


def test_dispatch_matches_reference_golden(orc, golden):
    for d in golden("dispatch.json"):
        a = matrix_recipe(d["a"], d["m"], d["k"], d["seed_a"])
        b = matrix_recipe(d["b"], d["k"], d["n"], d["seed_b"])
        rc, c, res = orc.dispatch_cgemm(a, b, O.make_config(**d["cfg"]))
        assert rc == d["rc"]
        assert res.line.decode() == d["line"], d
        assert (O.KINDS[res.kind], res.scale_a, res.scale_b) == (d["kind"], d["scale_a"], d["scale_b"])
        assert hashlib.sha256(bits(c.view(np.float32)).tobytes()).hexdigest() == d["c_bits_sha"]


def test_permute_matches_reference_golden(orc, golden):
    for case, d in golden("permute.json").items():
        t = matrix_recipe("uniform", 1, int(np.prod(d["dims"])), 700 + int(case)).reshape(d["dims"])
        out = orc.permute(t, d["axis"])
        assert bits(out.reshape(-1).view(np.float32)).tolist() == d["out"]
        assert np.array_equal(out, np.transpose(t, d["axis"]))


# -------------------------------------------------------------- networks
def test_circuit_text_and_path_match_reference_golden(golden):
    from oracle.network import greedy_path
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular, save_circuit
    for rq in golden("rqc.json"):
        c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
        assert save_circuit(c) == rq["circuit_text"]
        spec = circuit_to_network(c, [0] * c.n_qubits)
        assert [list(s) for s in greedy_path(spec)] == rq["path"]


@pytest.mark.parametrize("case", [0, 1, 2])
def test_network_oracle_matches_reference_amplitudes(golden, case):
    """The oracle's TTGT fold reproduces the reference amplitudes bit for bit in
    every FP32/FP64-tier mode (FP32 baseline, default AUTO-0 on small
    circuits), and within tolerance the f64 oracles."""
    from oracle.network import amplitude_sv, contract_network, contract_network_f64
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
    rq = golden("rqc.json")[case]
    c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
    for row in rq["amplitudes"][:4]:
        spec = circuit_to_network(c, row["x"])
        path = [tuple(s) for s in rq["path"]]
        for label, kw in (("BASELINE", dict(force="FP32_REF")), ("AUTO-0", dict()),
                          ("FP16TCEC", dict(force="FP16TCEC")), ("TF32TCEC", dict(force="TF32TCEC"))):
            _, _, z, _ = contract_network(spec, path, O.make_config(**kw))
            assert bits(z.view(np.float32)).tolist() == row[label], label
        _, _, z64 = contract_network_f64(spec, path)
        assert abs(complex(z64[0]) - complex(*row["tn_oracle"])) <= 1e-12 * max(abs(complex(*row["tn_oracle"])), 1e-30)
        sv = amplitude_sv(c, row["x"])
        assert abs(sv - complex(*row["sv_oracle"])) <= 1e-12


def test_workload_generator_is_the_reference_rng():
    """paper_2303_08989_b200.workload (the bench's configs[1] inputs) draws the
    same stream as rng.hpp's Rng: pinned against the oracle restatement and,
    where it is built, the reference's own ref_gemm_bench_operands."""
    import ctypes as C

    import oracle as O
    from paper_2303_08989_b200.workload import WorkloadRng, sweep_operands
    a, b = sweep_operands(96, pinned=False, m=40, k=72)
    r = O.Rng(1 + 96)
    assert np.array_equal(a.numpy().view(np.uint32), r.uniform_c32(40, 72).view(np.uint32))
    assert np.array_equal(b.numpy().view(np.uint32), r.uniform_c32(72, 96).view(np.uint32))
    g = WorkloadRng(5)
    o = O.Rng(5)
    assert [g.next_u64() for _ in range(5)] == [o.next_u64() for _ in range(5)]
    assert np.array_equal(WorkloadRng(9).gaussian(7, 1e-2), np.array(_gauss(9, 7)))
    ref = O.reference()
    if ref is not None:
        fa = np.empty((40, 72), np.complex64)
        fb = np.empty((72, 96), np.complex64)
        ref.lib.ref_gemm_bench_operands.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                                    C.c_void_p, C.c_void_p]
        ref.lib.ref_gemm_bench_operands(1 + 96, 40, 72, 96, fa.ctypes.data, fb.ctypes.data)
        assert np.array_equal(a.numpy().view(np.uint32), fa.view(np.uint32))
        assert np.array_equal(b.numpy().view(np.uint32), fb.view(np.uint32))


def _gauss(seed, n):
    import oracle as O
    r = O.Rng(seed)
    return [r.gaussian(1e-2) for _ in range(n)]


def test_network_text_format_matches_the_reference(golden):
    """save_network (network.cpp:440-458) of the reference's circuit networks is
    byte-identical to the reference's own text (golden sha), and load_network
    round-trips it exactly."""
    import hashlib

    from paper_2303_08989_b200.circuits import circuit_to_network, load_circuit
    from paper_2303_08989_b200.network import load_network, save_network
    for case in golden("rqc.json"):
        circ = load_circuit(case["circuit_text"])
        spec = circuit_to_network(circ, [0] * circ.n_qubits)
        text = save_network(spec)
        assert hashlib.sha256(text.encode()).hexdigest() == case["network_text_sha"]
        back = load_network(text)
        assert back.labels == [list(map(str, l)) for l in spec.labels]
        assert back.dims == [list(d) for d in spec.dims]
        for x, y in zip(back.data, spec.data):
            assert np.array_equal(np.asarray(x).reshape(-1).view(np.uint32),
                                  np.asarray(y, np.complex64).reshape(-1).view(np.uint32))
