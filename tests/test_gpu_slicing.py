"""Sliced contraction across ranks with the DEVICE evaluator:
two processes share the one GPU of the test box (gloo for the all_gather --
the NCCL path needs one GPU per rank), each contracts its round-robin share
of the slices through the captured-graph node batch, and the slice-ordered
f64 sum is bit-identical to one rank evaluating every slice."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _plan():
    from oracle.network import greedy_path
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.slicing import SlicePlan, find_slices
    c = rqc_rectangular(4, 4, 10, 5)
    spec = circuit_to_network(c, [(q * 3) % 2 for q in range(c.n_qubits)])
    path = greedy_path(spec)
    return SlicePlan.build(spec, path, find_slices(spec, path, n_labels=5))


def _device_amp(plan, rank, world, cfg_kw):
    from paper_2303_08989_b200 import Handle, make_config
    from paper_2303_08989_b200.network import Network
    from paper_2303_08989_b200.slicing import device_evaluator, sliced_amplitude
    h = Handle(0)
    net = Network(h, plan.base)
    from paper_2303_08989_b200 import SelectionPolicy
    cfg = make_config(SelectionPolicy(**cfg_kw)) if cfg_kw else make_config()
    amp, full = sliced_amplitude(device_evaluator(net, plan, cfg, chunk=8),
                                 plan, rank, world)
    net.close()
    h.close()
    return amp, full


def _worker(rank, world, port, cfg_kw, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        amp, full = _device_amp(_plan(), rank, world, cfg_kw)
        q.put((rank, amp, full.tobytes(), None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, repr(e)))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg_kw", [{}, {"size_auto": 16, "size_tf32": 8}])
def test_two_ranks_on_device_match_one_rank_bitwise(cfg_kw):
    from oracle.network import contract_network_f64
    plan = _plan()
    assert plan.n_slices == 32
    amp1, full1 = _device_amp(plan, 0, 1, cfg_kw)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg_kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, amp, full, err in res:
        assert err is None, err
        assert amp == amp1
        assert full == full1.tobytes()
    # and the sum is the amplitude (f64 oracle of the unsliced network)
    _, _, z = contract_network_f64(plan.spec, plan.path)
    assert abs(amp1 - complex(z[0])) <= 1e-4 * abs(complex(z[0]))
