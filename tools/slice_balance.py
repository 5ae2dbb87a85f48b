"""Load balance of the sliced Sycamore contraction over W ranks, measured on ONE
GPU: every rank's round-robin share of the slices (slicing.rank_slices) is
timed in turn, and the per-rank maximum is what a W-GPU run (one process per
GPU, no data-path communication, one 8-byte-per-slice all_gather) would take.
This is a load-balance measurement, not a multi-GPU run.

    python tools/slice_balance.py [cycles] [W...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402
from paper_2303_08989_b200.slicing import SlicePlan, rank_slices  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 12
worlds = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
circ = sycamore_like(cyc, 1)
spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
path, sliced, kind = bench.load_or_build_plan(spec, cyc, "plan")
plan = SlicePlan.build(spec, path, sliced)
h = Handle(0)
net = Network(h, plan.base)
cfg = make_config()
net.node_batch(plan.path, plan.var, [plan.run_data(0)], cfg)  # capture / warm
t1 = None
for W in worlds:
    per_rank = []
    for r in range(W):
        ids = rank_slices(plan.n_slices, r, W)
        runs = [plan.run_data(i) for i in ids]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        net.node_batch(plan.path, plan.var, runs, cfg)
        torch.cuda.synchronize()
        per_rank.append(time.perf_counter() - t0)
    tmax = max(per_rank)
    t1 = t1 or tmax * W / worlds[0] if W == worlds[0] else t1
    print(f"W={W}: {plan.n_slices} slices, {plan.n_slices // W}-{-(-plan.n_slices // W)} per rank, "
          f"max rank time {tmax * 1e3:.1f} ms, min {min(per_rank) * 1e3:.1f} ms, "
          f"speedup vs W=1 {t1 / tmax:.2f}x", flush=True)
