"""Device-resident TTGT contraction and RCS amplitudes (reference
test_tensor.cpp:77-174, test_qcircuit.cpp:221-241, test_experiments.cpp:72-96).

FP32-tier contractions (every step of the 4x4 circuits under the default
policy) are bit-identical to the reference amplitudes in tests/golden/rqc.json."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle.network import amplitude_sv, contract_network as oracle_fold
from paper_2303_08989_b200 import ExtentMismatch, InvalidPath, SelectionPolicy, make_config
from paper_2303_08989_b200.circuits import (NetworkSpec, bitstrings_for, circuit_to_network,
                                            rqc_rectangular)
from paper_2303_08989_b200.network import Network, Tensor, amplitude, contract_pair
from tests.conftest import bits
from tests.golden.recipes import matrix_recipe

pytestmark = pytest.mark.gpu

BASELINE = make_config(force="FP32_REF")


def _t(labels, dims, seed):
    return Tensor(labels, dims, matrix_recipe("uniform", 1, int(np.prod(dims)), seed).reshape(-1))


def test_contract_pair_basics(handle):
    a = Tensor(["s"], [2], np.array([1, 0], np.complex64))
    b = Tensor(["s"], [2], np.array([1, 1], np.complex64))
    c = contract_pair(handle, a, b, BASELINE)
    assert c.labels == [] and c.data[0] == 1
    with pytest.raises(ExtentMismatch):
        contract_pair(handle, Tensor(["s"], [2], np.zeros(2, np.complex64)),
                      Tensor(["s"], [3], np.zeros(3, np.complex64)), BASELINE)
    t = _t(["a", "b", "c"], [3, 4, 5], 1)
    eye = Tensor(["c", "c2"], [5, 5], np.eye(5, dtype=np.complex64).reshape(-1))
    r = contract_pair(handle, t, eye, BASELINE)
    assert r.labels == ["a", "b", "c2"] and np.array_equal(bits(r.data.view(np.float32)),
                                                           bits(t.data.view(np.float32)))
    x, y = _t(["x"], [3], 2), _t(["y"], [2], 3)
    r = contract_pair(handle, x, y, BASELINE)
    assert r.dims == [3, 2]
    assert np.allclose(r.data.reshape(3, 2), np.outer(x.data, y.data), atol=1e-7)


@pytest.mark.parametrize("mode", ["FP32_REF", "TF32TCEC", "FP16TCEC"])
def test_contract_pair_random_vs_einsum(handle, mode):
    g = np.random.default_rng(2)
    for it in range(10):
        a = _t(["i", "j", "k"], [4, 4, 4], 100 + it)
        b = _t(["k", "l", "m"], [4, 4, 4], 200 + it)
        want = np.einsum("ijk,klm->ijlm", a.data.reshape(4, 4, 4).astype(np.complex128),
                         b.data.reshape(4, 4, 4).astype(np.complex128))
        got = contract_pair(handle, a, b, make_config(force=mode))
        assert got.labels == ["i", "j", "l", "m"]
        err = np.linalg.norm(got.data - want.reshape(-1)) / np.linalg.norm(want)
        assert err <= 1e-6, (mode, err)


def test_contraction_matches_oracle_fold_bit_exact_fp32_tier(handle):
    """Every FP32-tier step is bit-identical, so the whole fold is."""
    spec = NetworkSpec(labels=[["a", "b", "c"], ["c", "d"], ["d", "e", "a"], ["b", "e"]],
                       dims=[[3, 4, 5], [5, 6], [6, 2, 3], [4, 2]],
                       data=[matrix_recipe("uniform", 1, n, 40 + i).reshape(-1)
                             for i, n in enumerate((60, 30, 36, 8))])
    net = Network(handle, spec)
    for path in ([(0, 1), (2, 4), (3, 5)], [(2, 3), (0, 4), (1, 5)], [(0, 3), (1, 2), (4, 5)]):
        got, lines = net.contract(path, BASELINE, want_log=True)
        _, _, want, want_lines = oracle_fold(spec, path, O.make_config(force="FP32_REF"))
        assert np.array_equal(bits(got.data.view(np.float32)), bits(want.view(np.float32)))
        assert lines == want_lines


def test_path_errors(handle):
    spec = NetworkSpec(labels=[["a"], ["a", "b"], ["b"]], dims=[[2], [2, 2], [2]],
                       data=[np.ones(2, np.complex64), np.ones(4, np.complex64), np.ones(2, np.complex64)])
    net = Network(handle, spec)
    with pytest.raises(InvalidPath):
        net.contract([(0, 0)], BASELINE)
    with pytest.raises(InvalidPath):
        net.contract([(0, 1)], BASELINE)  # leaves two nodes
    with pytest.raises(InvalidPath):
        net.contract([(0, 1), (0, 2)], BASELINE)  # dead node


@pytest.fixture(params=[1, 2, 3], ids=["per-step", "fused", "hybrid"])
def executor(request, handle):
    handle.set_executor(request.param)
    yield request.param
    handle.set_executor(0)


@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_rqc_amplitudes_bit_exact_vs_reference(handle, golden, case, executor):
    rq = golden("rqc.json")[case]
    c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
    path = [tuple(s) for s in rq["path"]]
    for row in rq["amplitudes"]:
        net = Network(handle, circuit_to_network(c, row["x"]))
        assert [list(s) for s in net.greedy_path()] == rq["path"]
        for label, cfg in (("BASELINE", BASELINE), ("AUTO-0", make_config())):
            z = net.contract(path, cfg).data[0]
            assert bits(np.array([z.real, z.imag], np.float32)).tolist() == row[label], label
        net.close()


@pytest.mark.parametrize("case", [1, 2, 3])
def test_rqc_tensor_core_modes_accuracy(handle, golden, case):
    """TCEC modes vs the f64 state vector: median error <= 1e-4,
    within 4x of the CPU BASELINE median; FP16TC markedly worse."""
    rq = golden("rqc.json")[case]
    c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
    path = [tuple(s) for s in rq["path"]]
    errs = {m: [] for m in ("FP16TCEC", "TF32TCEC", "FP16TC", "AUTO-lowered")}
    base = []
    for row in rq["amplitudes"]:
        ref = complex(*row["sv_oracle"])
        net = Network(handle, circuit_to_network(c, row["x"]))
        for m in ("FP16TCEC", "TF32TCEC", "FP16TC"):
            z = complex(net.contract(path, make_config(force=m)).data[0])
            errs[m].append(abs(z - ref) / abs(ref))
        z, lines = net.contract(path, make_config(SelectionPolicy(size_auto=4, size_tf32=2)),
                                want_log=True)
        errs["AUTO-lowered"].append(abs(complex(z.data[0]) - ref) / abs(ref))
        if row is rq["amplitudes"][0]:
            # shapes of every dispatched GEMM are the reference's; decisions are
            # identical up to and including the first tensor-core step (its
            # operands are still bit-identical; later statistics see values the
            # tensor cores rounded differently from the CPU emulation)
            want = row["log_lowered"]
            assert [ln.split(",")[:3] for ln in lines] == [ln.split(",")[:3] for ln in want]
            first_tc = next((i for i, ln in enumerate(want)
                             if ln.split(",")[3] != "FP32_BASELINE"), len(want) - 1)
            assert lines[:first_tc + 1] == want[:first_tc + 1]
        bz = np.array(row["BASELINE"], np.uint32).view(np.float32)
        base.append(abs(complex(bz[0], bz[1]) - ref) / abs(ref))
        net.close()
    med = {k: float(np.median(v)) for k, v in errs.items()}
    mb = float(np.median(base))
    for m in ("FP16TCEC", "TF32TCEC", "AUTO-lowered"):
        assert med[m] <= 1e-4 and med[m] <= max(4 * mb, 1e-6), (m, med, mb)


def test_selector_batch_equals_single_amplitudes(handle, golden, executor):
    rq = golden("rqc.json")[2]  # 4x4, depth 1+8+1
    c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
    xs = [row["x"] for row in rq["amplitudes"]]
    net = Network(handle, circuit_to_network(c, xs[0]))
    path = [tuple(s) for s in rq["path"]]
    for cfg, label in ((BASELINE, "BASELINE"), (make_config(), "AUTO-0")):
        amps = net.selector_batch(path, xs, cfg)
        for z, row in zip(amps, rq["amplitudes"]):
            assert bits(np.array([z.real, z.imag], np.float32)).tolist() == row[label]
    net.close()


def test_selector_batch_pinned_out_and_batch_profile(handle, golden):
    """selector_batch into a caller-provided (pinned) output array gives the
    same bits; tcec_profile_read_batches counts each batch with a positive
    device time while profiling is on, and nothing after it is switched off."""
    import torch
    rq = golden("rqc.json")[2]
    c = rqc_rectangular(rq["rows"], rq["cols"], rq["depth"], rq["seed"])
    xs = np.array([row["x"] for row in rq["amplitudes"]], np.uint8)
    net = Network(handle, circuit_to_network(c, list(xs[0])))
    path = [tuple(s) for s in rq["path"]]
    want = net.selector_batch(path, xs, BASELINE)
    pin_bits = torch.empty(xs.shape, dtype=torch.uint8, pin_memory=True).numpy()
    pin_bits[...] = xs
    out = torch.empty(len(xs), dtype=torch.complex64, pin_memory=True).numpy()
    handle.profile(True)
    got = net.selector_batch(path, pin_bits, BASELINE, out=out)
    net.selector_batch(path, pin_bits, BASELINE, out=out)
    ms, count = handle.profile_read_batches()
    handle.profile(False)
    assert got is out and np.array_equal(out.view(np.uint32), want.view(np.uint32))
    assert count == 2 and ms > 0
    net.selector_batch(path, pin_bits, BASELINE, out=out)
    assert handle.profile_read_batches()[1] == 0  # profile(False) resets and stops counting
    with pytest.raises(ValueError):
        net.selector_batch(path, pin_bits, BASELINE, out=np.empty(3, np.complex64))
    net.close()


def test_amplitude_api_and_statevector(handle):
    c = rqc_rectangular(2, 3, 6, 21)
    g = np.random.default_rng(99)
    for _ in range(6):
        x = [int(v) for v in g.integers(0, 2, 6)]
        got = complex(amplitude(handle, c, x, SelectionPolicy()))
        want = amplitude_sv(c, x)
        assert abs(got - want) <= 1e-5 * abs(want)


def test_fused_and_per_step_agree_on_all_amplitudes_of_a_small_circuit(handle):
    """Every 2^9 amplitude of a 3x3 circuit: the two executors give the same
    bits and the probabilities sum to 1 (the circuit is unitary)."""
    c = rqc_rectangular(3, 3, 8, 7)
    xs = [[(v >> q) & 1 for q in range(9)] for v in range(512)]
    net = Network(handle, circuit_to_network(c, xs[0]))
    path = net.greedy_path()
    handle.set_executor(2)
    fused = net.selector_batch(path, xs, BASELINE)
    handle.set_executor(1)
    stepwise = net.selector_batch(path, xs, BASELINE)
    handle.set_executor(0)
    net.close()
    assert np.array_equal(fused.view(np.uint32), stepwise.view(np.uint32))
    assert abs(float(np.sum(np.abs(fused.astype(np.complex128)) ** 2)) - 1.0) < 1e-5


def test_sliced_amplitude_on_device(handle):
    from oracle.network import contract_network_f64
    from paper_2303_08989_b200.slicing import (SlicePlan, device_evaluator, find_slices,
                                               sliced_amplitude)
    c = rqc_rectangular(3, 4, 8, 11)
    spec = circuit_to_network(c, [1, 0] * 6)
    path = Network(None, spec).greedy_path()
    _, _, z = contract_network_f64(spec, path)
    plan = SlicePlan.build(spec, path, find_slices(spec, path, n_labels=4))
    net = Network(handle, plan.base)
    for policy in (1, 2, 3):
        handle.set_executor(policy)
        amp, full = sliced_amplitude(device_evaluator(net, plan, BASELINE), plan)
        assert abs(amp - complex(z[0])) <= 1e-5 * abs(complex(z[0]))
    handle.set_executor(0)
    net.close()


@pytest.mark.parametrize("seed", [3, 8])
def test_hybrid_subtree_launch_matches_per_step_with_tensor_core_steps(handle, seed):
    """Lowered size thresholds put the larger steps of a 5x5 network on the
    tensor-core tiers, so the whole-network fused path is ineligible and the
    auto / hybrid executors run the tiny SIMT subtrees in one launch before the
    per-step graph: results must be bit-identical to the pure per-step fold
    (single contraction, selector batch replays and node batches)."""
    c = rqc_rectangular(5, 5, 12, seed)
    xs = [[(v * 2654435761 >> q) & 1 for q in range(25)] for v in range(6)]
    net = Network(handle, circuit_to_network(c, xs[0]))
    path = net.greedy_path()
    cfg = make_config(SelectionPolicy(size_auto=16, size_tf32=4))
    out = {}
    for policy in (1, 3, 0):
        handle.set_executor(policy)
        single, log = net.contract(path, cfg, want_log=True)
        batch = net.selector_batch(path, xs, cfg)
        out[policy] = (single.data.view(np.uint32).copy(), batch.view(np.uint32).copy(), log)
    handle.set_executor(0)
    net.close()
    assert any("TF32" in line or "FP16" in line for line in out[1][2]), "no tensor-core step"
    for policy in (3, 0):
        assert np.array_equal(out[policy][0], out[1][0]), policy
        assert np.array_equal(out[policy][1], out[1][1]), policy
        assert out[policy][2] == out[1][2]


def test_thread_per_run_batch_matches_warp_per_run(handle):
    """From 4096 runs the fused program runs one thread per bitstring over a
    structure-of-arrays arena; the same per-element chains as the
    warp-per-bitstring kernel (itself pinned to the reference above) ->
    bit-identical amplitudes, selectors and node-data batches alike."""
    circ = rqc_rectangular(4, 4, 8, 1)
    allx = np.array([[(v >> q) & 1 for q in range(16)] for v in range(1 << 16)], np.uint8)
    xs = allx[::7][:6144]
    net = Network(handle, circuit_to_network(circ, xs[0]))
    path = net.greedy_path()
    cfg = make_config()
    big = net.selector_batch(path, xs, cfg)                        # thread per run
    small = np.concatenate([net.selector_batch(path, xs[i:i + 2048], cfg)  # warp per run
                            for i in range(0, len(xs), 2048)])
    assert np.array_equal(big.view(np.uint32), small.view(np.uint32))
    net.close()


def test_device_f64_oracle_is_the_reference_oracle(handle, golden):
    """tcec_contract_network_oracle (the f64 TTGT fold on the device) equals the
    reference's own contract_network_oracle (network.cpp:179-186) bit for bit:
    the golden `tn_oracle` amplitudes were computed by the unmodified reference
    along its greedy path for every golden circuit and bitstring (numpy's zgemm
    would not match: the reference sums four real planes in ascending k)."""
    from paper_2303_08989_b200.circuits import circuit_to_network, load_circuit
    from paper_2303_08989_b200.network import Network
    checked = 0
    for case in golden("rqc.json"):
        circ = load_circuit(case["circuit_text"])
        path = [tuple(p) for p in case["path"]]
        for row in case["amplitudes"]:
            net = Network(handle, circuit_to_network(circ, row["x"]))
            z = complex(net.contract_oracle(path).data.reshape(-1)[0])
            net.close()
            assert (z.real, z.imag) == tuple(row["tn_oracle"]), (case["rows"], case["cols"], row["x"])
            checked += 1
    assert checked >= 40


@pytest.mark.parametrize("depth", [12, 14])
def test_rqc7x7_tensor_core_amplitudes(handle, depth):
    """configs[4]: 7x7 RQC at depth 12 / 14 on the reference's greedy path with
    a lowered policy that routes the large steps to the tensor-core tiers --
    median amplitude error vs the f64 contraction oracle <= 1e-4 and <= 4x the
    FP32 baseline tier's (experiments.cpp:240-256)."""
    from paper_2303_08989_b200 import SelectionPolicy, make_config
    from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.network import Network
    circ = rqc_rectangular(7, 7, depth, 1)
    xs = bitstrings_for(49, 10, 1)[:4]
    spec = circuit_to_network(circ, xs[0])
    net = Network(handle, spec)
    path = net.greedy_path()
    ref = []
    for x in xs:
        n2 = Network(handle, circuit_to_network(circ, x))
        ref.append(complex(n2.contract_oracle(path).data.reshape(-1)[0]))
        n2.close()
    ref = np.array(ref)
    auto = make_config(SelectionPolicy(size_auto=256, size_tf32=64))
    _, lines = net.contract(path, auto, want_log=True)
    kinds = {ln.split(",")[3] for ln in lines}
    assert kinds & {"TF32TCEC", "FP16TCEC", "FP16TCEC_SCALED"}, kinds
    z_auto = net.selector_batch(path, xs, auto).astype(np.complex128)
    z_fp32 = net.selector_batch(path, xs, make_config(force="FP32_REF")).astype(np.complex128)
    net.close()
    e_auto = np.median(np.abs(z_auto - ref) / np.abs(ref))
    e_fp32 = np.median(np.abs(z_fp32 - ref) / np.abs(ref))
    assert e_auto <= 1e-4, (e_auto, kinds)
    assert e_auto <= 4 * e_fp32, (e_auto, e_fp32, kinds)


def test_device_statevector_is_the_reference_oracle(handle, golden):
    """tcec_statevector_f64 == the reference's statevector_oracle bit for bit
    (golden `sv_oracle` amplitudes computed by the unmodified reference)."""
    from paper_2303_08989_b200.circuits import load_circuit
    from paper_2303_08989_b200.network import statevector_oracle
    checked = 0
    for case in golden("rqc.json"):
        circ = load_circuit(case["circuit_text"])
        sv = statevector_oracle(handle, circ).cpu().numpy()
        for row in case["amplitudes"]:
            idx = sum(int(b) << q for q, b in enumerate(row["x"]))
            z = sv[idx]
            assert (z.real, z.imag) == tuple(row["sv_oracle"]), (case["rows"], case["cols"], row["x"])
            checked += 1
    assert checked >= 40


def _skinny_chain(seed, t_dims, gates):
    """A big tensor T contracted with a chain of small tensors on scattered
    axes -- the skinny FP32-tier steps of sliced RCS contractions.  gates:
    (number of T axes contracted, new axis extents, T first?)."""
    g = np.random.default_rng(seed)
    labels = [[f"t{i}" for i in range(len(t_dims))]]
    dims = [list(t_dims)]
    cur = list(zip(labels[0], t_dims))
    path, nxt = [], 1 + len(gates)
    prev = 0
    for gi, (nk, new_dims, t_first) in enumerate(gates):
        pick = sorted(g.choice(len(cur), size=nk, replace=False), key=lambda _: g.random())
        shared = [cur[i] for i in pick]
        new = [(f"n{gi}_{j}", d) for j, d in enumerate(new_dims)]
        gl = [l for l, _ in shared] + [l for l, _ in new]
        gd = [d for _, d in shared] + [d for _, d in new]
        order = g.permutation(len(gl))
        labels.append([gl[i] for i in order])
        dims.append([gd[i] for i in order])
        path.append((prev, gi + 1) if t_first else (gi + 1, prev))
        keep = [c for c in cur if c not in shared]
        cur = keep + new if t_first else new + keep
        prev = nxt
        nxt += 1
    data = [matrix_recipe("uniform", 1, int(np.prod(d)), seed + 7 * i).reshape(-1) for i, d in enumerate(dims)]
    return NetworkSpec(labels=labels, dims=dims, data=data), path


@pytest.mark.parametrize("case", [
    ([2] * 16, [(2, [2, 2], False), (3, [2, 2, 2], False), (4, [2] * 4, True), (1, [2], True)]),
    ([2] * 18, [(4, [2] * 5, False), (3, [2] * 3, True), (2, [2] * 4, False)]),     # m = 32: two passes
    ([3, 2, 4, 2, 2, 5, 2, 2, 2, 2, 2, 3, 2, 2], [(2, [3, 2], False), (2, [5], True), (2, [2, 2], False)]),
    ([2] * 21, [(7, [2] * 3, False), (5, [2] * 2, True)]),                       # k = 128 / 32
])
@pytest.mark.parametrize("executor", [0, 1, 3], ids=["auto", "per-step", "hybrid"])
def test_skinny_view_gather_bit_exact(handle, case, executor):
    """Skinny FP32-tier steps read their long operand through a strided view of
    the unpermuted tensor (fused TTGT gather; col kernel when the long operand
    is B, row kernel when it is A; power-of-two and mixed extents): the fold
    equals the oracle's permute-then-GEMM fold bit for bit, decision lines
    included."""
    t_dims, gates = case
    spec, path = _skinny_chain(5 + len(t_dims), t_dims, gates)
    _, _, _, lines0 = oracle_fold(spec, path, O.make_config(force="FP32_REF"))
    for ln in lines0:  # every step takes the skinny kernels
        m, n, k = (int(v) for v in ln.split(",")[:3])
        assert k <= 128 and min(m, n) <= 32 and max(m, n) >= 4096, ln
    handle.set_executor(executor)
    net = Network(handle, spec)
    try:
        got, lines = net.contract(path, BASELINE, want_log=True)
        labels, _, want, want_lines = oracle_fold(spec, path, O.make_config(force="FP32_REF"))
        assert got.labels == labels
        assert np.array_equal(bits(got.data.view(np.float32)), bits(want.view(np.float32)))
        assert lines == want_lines
        got2, _ = net.contract(path, make_config(), want_log=True)
        _, _, want2, _ = oracle_fold(spec, path, O.make_config())
        assert np.array_equal(bits(got2.data.view(np.float32)), bits(want2.view(np.float32)))
    finally:
        net.close()
        handle.set_executor(0)


def _tc_view_spec(case):
    """Networks whose tensor-core steps need operand permutes (scrambled shared
    and free axes on both sides)."""
    if case == 0:    # one TF32-tier step (512 <= min < 2048), A-expanded layout (m < n)
        labels = [["x1", "s1", "x2", "s2"], ["s2", "y1", "s1", "y2"]]
        dims = [[16, 32, 32, 16], [16, 32, 32, 32]]
        path = [(0, 1)]
    elif case == 1:  # one AUTO step (min >= 2048), B-expanded layout (m > n)
        labels = [["s1", "x1", "s2", "x2"], ["y1", "s2", "s1"]]
        dims = [[64, 64, 32, 64], [2048, 32, 64]]
        path = [(0, 1)]
    else:            # a chain: the intermediate feeds a second permuted tensor-core step
        labels = [["x1", "s1", "x2", "s2"], ["s2", "y1", "s1", "y2"], ["y2", "z1", "x1", "z2"]]
        dims = [[16, 32, 32, 16], [16, 32, 32, 32], [32, 32, 16, 32]]
        path = [(0, 1), (2, 3)]
    data = [matrix_recipe("uniform", 1, int(np.prod(d)), 90 + i).reshape(-1) for i, d in enumerate(dims)]
    return NetworkSpec(labels=labels, dims=dims, data=data), path


_VIEW_OFF_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2303_08989_b200 import Handle, make_config
from paper_2303_08989_b200.network import Network
from tests.test_gpu_network import _tc_view_spec
spec, path = _tc_view_spec({case})
h = Handle(0)
net = Network(h, spec)
r, lines = net.contract(path, make_config(), want_log=True)
np.save({out!r}, r.data)
open({out!r} + ".log", "w").write("\\n".join(lines))
net.close(); h.close()
"""


@pytest.mark.parametrize("case", [0, 1, 2])
def test_tc_step_view_gather_bit_identical(handle, case, tmp_path):
    """Tensor-core steps read permuted operands through a strided view in the
    preparation kernels (fused TTGT gather; statistics on the unpermuted
    tensor): the contraction -- decision lines included -- is bit-identical to
    the permute-then-prepare path (TCEC_VIEW_GATHER=0 in a subprocess), and
    within the reference bar of the f64 oracle fold."""
    import os
    import subprocess
    import sys
    spec, path = _tc_view_spec(case)
    net = Network(handle, spec)
    try:
        got, lines = net.contract(path, make_config(), want_log=True)
        ref = net.contract_oracle(path).data
    finally:
        net.close()
    assert all(ln.split(",")[3] in ("TF32TCEC", "FP16TCEC", "FP16TCEC_SCALED") for ln in lines), lines
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "off.npy")
    env = dict(os.environ, TCEC_VIEW_GATHER="0")
    subprocess.run([sys.executable, "-c", _VIEW_OFF_SCRIPT.format(root=root, case=case, out=out)],
                   env=env, cwd=root, check=True, timeout=600)
    off = np.load(out)
    assert open(out + ".log").read().split("\n") == lines
    assert np.array_equal(bits(got.data.view(np.float32)), bits(off.view(np.float32)))
    err = np.linalg.norm(got.data.astype(np.complex128) - ref) / np.linalg.norm(ref)
    assert err <= 5e-6, err


def _random_network(rng, seed):
    """Random connected tensor network: 4-7 tensors of rank <= 5, bonds of
    extent 1-5 (size-1 and repeated extents included), a few open legs."""
    nt = int(rng.integers(4, 8))
    labels = [[] for _ in range(nt)]
    dims = [[] for _ in range(nt)]
    nb = 0

    def bond(i, j, d):
        nonlocal nb
        nm = f"b{nb}"
        nb += 1
        labels[i].append(nm)
        dims[i].append(d)
        labels[j].append(nm)
        dims[j].append(d)

    for i in range(1, nt):  # connected: a random tree, then extra bonds
        bond(int(rng.integers(0, i)), i, int(rng.integers(1, 6)))
    for _ in range(int(rng.integers(1, 5))):
        i, j = (int(x) for x in rng.choice(nt, 2, replace=False))
        if len(labels[i]) < 5 and len(labels[j]) < 5:
            bond(i, j, int(rng.integers(1, 6)))
    for o in range(int(rng.integers(0, 3))):
        i = int(rng.integers(0, nt))
        labels[i].append(f"o{o}")
        dims[i].append(int(rng.integers(1, 4)))
    for i in range(nt):  # random axis order per tensor
        perm = rng.permutation(len(labels[i]))
        labels[i] = [labels[i][p] for p in perm]
        dims[i] = [dims[i][p] for p in perm]
    data = [matrix_recipe("uniform", 1, int(np.prod(d)) if d else 1, seed * 31 + i).reshape(-1)
            for i, d in enumerate(dims)]
    return NetworkSpec(labels=labels, dims=dims, data=data)


def _random_path(rng, n):
    live, nxt, path = list(range(n)), n, []
    while len(live) > 1:
        a, b = (int(x) for x in rng.choice(len(live), 2, replace=False))
        ia, ib = live[a], live[b]
        path.append((ia, ib))
        live = [x for x in live if x not in (ia, ib)] + [nxt]
        nxt += 1
    return path


@pytest.mark.parametrize("executor", [0, 1, 3])
def test_random_networks_fp32_tier_bit_exact_vs_oracle_fold(handle, executor):
    """Random networks and random contraction orders (ragged extents, size-1
    bonds, open legs, shuffled axes -> every TTGT permute / fused-gather case
    of small tensors) through each executor: the FP32 tier is bit-identical to
    the oracle fold (network.cpp:149-177) and the decision-log lines match."""
    rng = np.random.default_rng(90 + executor)
    handle.set_executor(executor)
    try:
        for case in range(12):
            spec = _random_network(rng, 100 * executor + case)
            path = _random_path(rng, len(spec.labels))
            net = Network(handle, spec)
            got, lines = net.contract(path, BASELINE, want_log=True)
            net.close()
            wl, wd, want, want_lines = oracle_fold(spec, path, O.make_config(force="FP32_REF"))
            assert list(got.labels) == list(wl), (case, got.labels, wl)
            assert np.array_equal(bits(got.data.view(np.float32)), bits(np.asarray(want).view(np.float32))), case
            assert lines == want_lines, case
    finally:
        handle.set_executor(0)
