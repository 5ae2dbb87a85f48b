"""Contraction-path and slice search (host logic, CPU):
every path the search returns is a valid SSA fold of the reference's network
(network.cpp:149-168) whose f64 oracle contraction equals the greedy path's
amplitude; reconfiguration never raises the modelled cost; the sliced plan's
slice sum equals the unsliced amplitude; the cost bookkeeping matches an
independent recount."""
import math

import numpy as np
import pytest

from oracle.network import contract_network_f64, greedy_path
from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular, sycamore_like
from paper_2303_08989_b200.paths import (hyper_path, model_step_cost, partition_path,
                                         path_cost, path_model_cost, presimplify,
                                         random_greedy_path, reconfigure_path, remap_path)
from paper_2303_08989_b200.slicing import SlicePlan, assignment, slice_spec


def _rqc(rows=3, cols=4, depth=8, seed=5):
    c = rqc_rectangular(rows, cols, depth, seed)
    return circuit_to_network(c, [(q * 3 + 1) % 2 for q in range(c.n_qubits)])


def _syc(cycles=2):
    c = sycamore_like(cycles, 1)
    return circuit_to_network(c, [(q * 7 + 3) % 2 for q in range(c.n_qubits)])


def _valid_ssa(spec, path):
    live = set(range(len(spec.labels)))
    nxt = len(spec.labels)
    for a, b in path:
        assert a != b and a in live and b in live
        live -= {a, b}
        live.add(nxt)
        nxt += 1
    assert len(live) == 1


def _amp(spec, path):
    _, _, z = contract_network_f64(spec, path)
    return complex(np.asarray(z).reshape(-1)[0])


@pytest.mark.parametrize("maker", [_rqc, _syc])
def test_presimplify_then_partition_is_a_valid_equal_path(maker):
    spec = maker()
    ref = _amp(spec, greedy_path(spec))
    pre, ids, red = presimplify(spec)
    # every survivor of rank <= 2 is isolated (e.g. a qubit no gate touched)
    for i, ls in enumerate(red.labels):
        if len(ls) <= 2:
            assert not any(set(ls) & set(o) for j, o in enumerate(red.labels) if j != i)
    p, f, w = partition_path(red, trials=2, leaf=8)
    full = remap_path(pre, ids, len(spec.labels), p)
    _valid_ssa(spec, full)
    z = _amp(spec, full)
    assert abs(z - ref) <= 1e-9 * max(abs(ref), 1e-30)


@pytest.mark.parametrize("native", [True, False])
def test_reconfigure_never_raises_cost_and_keeps_the_value(native):
    """Both the native C++ engine (tcec_path_reconfigure, host code in the
    library -- no GPU needed) and the Python restatement."""
    spec = _rqc(3, 4, 10)
    pre, ids, red = presimplify(spec)
    p, _, _ = random_greedy_path(red, trials=2, max_width=40)
    for tm in (False, True):
        before = path_model_cost(red, p, (), tm)
        q, f, w = reconfigure_path(red, p, k=8, passes=2, time_model=tm, native=native)
        _valid_ssa(red, q)
        assert path_model_cost(red, q, (), tm) <= before * (1 + 1e-9)
        full_p = remap_path(pre, ids, len(spec.labels), p)
        full_q = remap_path(pre, ids, len(spec.labels), q)
        assert abs(_amp(spec, full_q) - _amp(spec, full_p)) <= 1e-9 * abs(_amp(spec, full_p))


def test_hyper_path_slices_to_the_width_and_sums_back():
    spec = _rqc(3, 3, 8)
    ref = _amp(spec, greedy_path(spec))
    _, _, w0 = hyper_path(spec, max_log2=60.0, trials=1)[1:]
    target = max(2.0, w0 - 2.0)
    path, sliced, flops, width = hyper_path(spec, max_log2=target, trials=1)
    _valid_ssa(spec, path)
    assert width <= target and len(sliced) >= 1
    plan = SlicePlan.build(spec, path, sliced)
    total = 0j
    for i in range(plan.n_slices):
        total += _amp(slice_spec(spec, plan.sliced, assignment(i, plan.dims)), path)
    assert abs(total - ref) <= 1e-9 * abs(ref)


def test_path_cost_matches_an_independent_recount():
    spec = _rqc(3, 3, 6)
    path = greedy_path(spec)
    flops, width = path_cost(spec, path)
    dims = {l: d for ls, ds in zip(spec.labels, spec.dims) for l, d in zip(ls, ds)}
    live = {i: list(ls) for i, ls in enumerate(spec.labels)}
    nxt, f2, w2 = len(spec.labels), 0.0, 0.0
    for a, b in path:
        la, lb = live.pop(a), live.pop(b)
        out = [l for l in la if l not in lb] + [l for l in lb if l not in la]
        k = math.prod(dims[l] for l in la if l in lb)
        f2 += 8.0 * math.prod(dims[l] for l in out) * k
        w2 = max(w2, math.log2(max(1, math.prod(dims[l] for l in out))))
        live[nxt] = out
        nxt += 1
    assert flops == pytest.approx(f2) and width == pytest.approx(w2)


def test_model_cost_tiers_and_latency():
    # same MACs: a TF32-tier shape (min 512) is modelled cheaper than a SIMT one
    simt = model_step_cost(9 + 8, 8 + 10, 9 + 10)     # m=512, n=1024, k=256
    tc = model_step_cost(9 + 9, 9 + 9, 18)            # m=n=k=512
    assert tc < simt
    # a 16-output, 2^21-long step pays the chain latency
    assert model_step_cost(2 + 21, 2 + 21, 4) > 1e3 * 2.0 ** 25 / 1e2


def test_native_and_python_reconfigure_agree_on_cost():
    spec = _syc(4)
    pre, ids, red = presimplify(spec)
    p, _, _ = random_greedy_path(red, trials=1, max_width=60)
    qn, _, _ = reconfigure_path(red, p, k=8, passes=2, native=True, time_model=True)
    qp, _, _ = reconfigure_path(red, p, k=8, passes=2, native=False, time_model=True)
    cn, cp = path_model_cost(red, qn, (), True), path_model_cost(red, qp, (), True)
    assert cn <= path_model_cost(red, p, (), True) and cp <= path_model_cost(red, p, (), True)
    assert cn == pytest.approx(cp, rel=0.25)
