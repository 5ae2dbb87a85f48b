"""Slice finder / scheduler / cross-rank sum (host logic, CPU) -- the sliced
amplitude equals the unsliced one, per-slice values come from the f64 oracle
contraction, and the world-size-2 gloo run reproduces the world-size-1 result
bit for bit (one all_gather, slice-ordered float64 sum)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle.network import contract_network_f64, greedy_path
from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
from paper_2303_08989_b200.slicing import (SlicePlan, contraction_cost, find_slices,
                                           rank_slices, slice_spec, sliced_amplitude)


def _spec(rows=3, cols=3, depth=6, seed=3, x=None):
    c = rqc_rectangular(rows, cols, depth, seed)
    x = x or [q % 2 for q in range(c.n_qubits)]
    spec = circuit_to_network(c, x)
    return spec, greedy_path(spec)


def _oracle_eval(plan):
    def ev(ids):
        out = []
        for i in ids:
            from paper_2303_08989_b200.slicing import assignment
            sub = slice_spec(plan.spec, plan.sliced, assignment(i, plan.dims))
            _, _, z = contract_network_f64(sub, plan.path)
            out.append(np.complex64(z[0]))
        return np.array(out, np.complex64)
    return ev


def test_find_slices_reduces_the_largest_intermediate():
    spec, path = _spec(3, 4, 8)
    big0, macs0 = contraction_cost(spec, path)
    sl = find_slices(spec, path, n_labels=3)
    assert len(sl) == 3 and len(set(sl)) == 3
    big, macs = contraction_cost(spec, path, sl)
    assert big <= big0 // 2
    assert find_slices(spec, path, n_labels=3) == sl  # deterministic
    assert max(len(find_slices(spec, path, max_elems=big0 // 4)), 0) >= 1


def test_sliced_sum_equals_unsliced_amplitude():
    spec, path = _spec()
    _, _, z = contract_network_f64(spec, path)
    sl = find_slices(spec, path, n_labels=4)
    plan = SlicePlan.build(spec, path, sl)
    assert plan.n_slices == 16
    amp, full = sliced_amplitude(_oracle_eval(plan), plan)
    assert abs(amp - complex(z[0])) <= 1e-6 * abs(complex(z[0]))


def test_round_robin_partition_covers_every_slice_once():
    for n in (1, 7, 16, 64):
        for w in (1, 2, 3, 8):
            ids = sorted(i for r in range(w) for i in rank_slices(n, r, w))
            assert ids == list(range(n))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec, path = _spec()
    plan = SlicePlan.build(spec, path, find_slices(spec, path, n_labels=4))
    amp, full = sliced_amplitude(_oracle_eval(plan), plan, rank, world)
    q.put((rank, amp, full.tobytes()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_matches_single_rank_bitwise():
    spec, path = _spec()
    plan = SlicePlan.build(spec, path, find_slices(spec, path, n_labels=4))
    amp1, full1 = sliced_amplitude(_oracle_eval(plan), plan)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, amp, full in res:
        assert amp == amp1
        assert full == full1.tobytes()


def test_run_data_equals_slice_spec_variable_nodes():
    """SlicePlan.run_data slices only the variable nodes; its arrays equal the
    variable nodes of the full slice_spec sub-network bit for bit, for every
    slice, and the other nodes of every slice equal the plan's base."""
    from paper_2303_08989_b200.slicing import assignment
    spec, path = _spec(3, 3, 6, 5)
    sliced = find_slices(spec, path, n_labels=3)
    plan = SlicePlan.build(spec, path, sliced)
    assert plan.n_slices > 1
    var = set(plan.var)
    for i in range(plan.n_slices):
        sub = slice_spec(plan.spec, plan.sliced, assignment(i, plan.dims))
        got = plan.run_data(i)
        assert len(got) == len(plan.var)
        for j, g in zip(plan.var, got):
            assert np.array_equal(g.view(np.uint32), sub.data[j].view(np.uint32))
        for j in range(len(sub.data)):
            if j not in var:
                assert np.array_equal(sub.data[j].view(np.uint32), plan.base.data[j].view(np.uint32))
