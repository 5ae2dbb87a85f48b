"""Device errors and decisions of batch contractions (selector / node batch):
every run's tensor-core decisions are archived on the device and read back
with the amplitudes, so a run that hits ScaleOverflow (precsel.cpp:54-57,
209-216) fails the batch naming the run, the FP16 saturation flag
(DispatchResult::overflow) is reported per run, and each run's decision-log
lines equal the single-contraction log of the same data (and the reference
restatement's), as amplitude(..., log) records them (qcircuit.cpp:184-195)."""
import numpy as np
import pytest

import oracle as O
from oracle.network import contract_network as oracle_fold
from paper_2303_08989_b200 import ScaleOverflow, SelectionPolicy, make_config
from paper_2303_08989_b200.circuits import NetworkSpec
from paper_2303_08989_b200.network import Network

pytestmark = pytest.mark.gpu

LOW = dict(size_auto=16, size_tf32=8)


def _chain(seed, dims=(64, 48, 40, 32)):
    """A - B - C chain: two contractions large enough for the statistics tier
    under the lowered policy."""
    r = np.random.default_rng(seed)
    a, b, c, d = dims

    def u(*s):
        return (r.uniform(-1, 1, s) + 1j * r.uniform(-1, 1, s)).astype(np.complex64)
    return NetworkSpec(labels=[["i", "j"], ["j", "k"], ["k", "l"]], dims=[[a, b], [b, c], [c, d]],
                       data=[u(a, b), u(b, c), u(c, d)])


def _runs(spec, var, n, seed, edit=None):
    r = np.random.default_rng(seed)
    out = []
    for i in range(n):
        run = []
        for v in var:
            x = (r.uniform(-1, 1, spec.data[v].shape) + 1j * r.uniform(-1, 1, spec.data[v].shape))
            x = x.astype(np.complex64)
            if edit:
                x = edit(i, v, x)
            run.append(x)
        out.append(run)
    return out


def _closed(spec):
    """close the chain with two vectors so the batch yields one value per run"""
    r = np.random.default_rng(7)
    li, ll = spec.dims[0][0], spec.dims[-1][-1]
    v1 = (r.uniform(-1, 1, li) + 1j * r.uniform(-1, 1, li)).astype(np.complex64)
    v2 = (r.uniform(-1, 1, ll) + 1j * r.uniform(-1, 1, ll)).astype(np.complex64)
    return NetworkSpec(labels=spec.labels + [["i"], ["l"]], dims=spec.dims + [[li], [ll]],
                       data=spec.data + [v1, v2])


PATH = [(0, 1), (5, 2), (6, 3), (7, 4)]  # (A B) C, then the two closing vectors


def test_scale_overflow_in_one_run_raises_naming_it(handle):
    spec = _closed(_chain(1))
    var = [0]

    def edit(i, v, x):
        if i == 2:
            x[:] = np.complex64(np.inf)  # e_max 128, r2 = 0 -> FP16TCEC_SCALED, s = -114 -> inf
        return x
    runs = _runs(spec, var, 4, 3, edit)
    net = Network(handle, spec)
    cfg = make_config(SelectionPolicy(**LOW))
    with pytest.raises(ScaleOverflow, match="run 2"):
        net.node_batch(PATH, var, runs, cfg)
    # the reference restatement throws ScaleOverflow on that run's data too
    sub = NetworkSpec(spec.labels, spec.dims, [runs[2][0]] + spec.data[1:])
    with pytest.raises(RuntimeError):
        oracle_fold(sub, PATH, O.make_config(**LOW))
    # clean runs still go through and agree with single contractions
    vals = net.node_batch(PATH, var, [runs[0], runs[1]], cfg)
    for i in range(2):
        s2 = NetworkSpec(spec.labels, spec.dims, [runs[i][0]] + spec.data[1:])
        n2 = Network(handle, s2)
        assert vals[i] == n2.contract(PATH, cfg).data[0]
        n2.close()
    net.close()


def test_fp16_overflow_flag_is_per_run(handle):
    spec = _closed(_chain(2))
    var = [1]

    def edit(i, v, x):
        if i == 1:
            x[3, 4] = np.complex64(1e6)  # past the FP16 maximum: saturates, flag set
        return x
    runs = _runs(spec, var, 3, 5, edit)
    net = Network(handle, spec)
    cfg = make_config(SelectionPolicy(**LOW), force="FP16TCEC")
    net.node_batch(PATH, var, runs, cfg)
    flags = [net.batch_run_info(r, len(PATH))[0] for r in range(3)]
    assert flags == [False, True, False]
    net.close()


@pytest.mark.parametrize("policy", [LOW, dict(size_auto=40, size_tf32=8), None])
def test_batch_decision_lines_match_single_contractions_and_oracle(handle, policy):
    spec = _closed(_chain(3))
    var = [0, 2]

    def edit(i, v, x):
        if i == 1 and v == 0:
            x *= np.float32(2.0 ** -20)   # -> FP16TCEC_SCALED for this run's first GEMM
        if i == 2 and v == 2:
            x[0, 0] = np.complex64(1.0)
            x[1:] *= np.float32(1e-9)       # wide exponent range -> TF32TCEC
        return x
    runs = _runs(spec, var, 3, 9, edit)
    net = Network(handle, spec)
    cfg = make_config(SelectionPolicy(**policy)) if policy else make_config()
    ocfg = O.make_config(**policy) if policy else O.make_config()
    net.node_batch(PATH, var, runs, cfg)
    kinds = set()
    for r in range(3):
        ovf, lines = net.batch_run_info(r, len(PATH))
        data = list(spec.data)
        for v, x in zip(var, runs[r]):
            data[v] = x
        s2 = NetworkSpec(spec.labels, spec.dims, data)
        n2 = Network(handle, s2)
        _, single = n2.contract(PATH, cfg, want_log=True)
        n2.close()
        _, _, _, olines = oracle_fold(s2, PATH, ocfg)
        assert lines == single, (r, lines, single)
        assert lines == olines, (r, lines, olines)
        kinds |= {ln.split(",")[3] for ln in lines}
    if policy == LOW:
        assert {"FP16TCEC_SCALED", "TF32TCEC"} <= kinds, kinds
    net.close()


def test_selector_batch_run_info(handle):
    """the selector batch archives decisions the same way (default executor on
    a circuit whose big steps reach the tensor-core tiers)"""
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
    circ = rqc_rectangular(4, 4, 8, 1)
    spec = circuit_to_network(circ, [0] * 16)
    net = Network(handle, spec)
    path = net.greedy_path()
    cfg = make_config(SelectionPolicy(size_auto=4, size_tf32=2))
    xs = [[(v >> q) & 1 for q in range(16)] for v in (0, 5, 77)]
    net.selector_batch(path, xs, cfg)
    for r, x in enumerate(xs):
        ovf, lines = net.batch_run_info(r, len(path))
        n2 = Network(handle, circuit_to_network(circ, x))
        _, single = n2.contract(path, cfg, want_log=True)
        n2.close()
        assert lines == single
        assert not ovf
    net.close()
