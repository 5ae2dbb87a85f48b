"""Host-side overhead of one sliced Sycamore amplitude on one GPU: slice data
generation, the node_batch call (wall) against its device batch time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402
from paper_2303_08989_b200.slicing import SlicePlan  # noqa: E402

circ = sycamore_like(12, 1)
spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
path, sliced, kind = bench.load_or_build_plan(spec, 12, "plan")
plan = SlicePlan.build(spec, path, sliced)
h = Handle(0)
net = Network(h, plan.base)
cfg = make_config()
runs = [plan.run_data(i) for i in range(plan.n_slices)]
net.node_batch(plan.path, plan.var, runs, cfg)
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    runs = [plan.run_data(i) for i in range(plan.n_slices)]
    t1 = time.perf_counter()
    h.profile(True)
    vals = net.node_batch(plan.path, plan.var, runs, cfg)
    t2 = time.perf_counter()
    dev_ms, nb = h.profile_read_batches()
    h.profile(False)
    print(f"run_data {1e3 * (t1 - t0):.1f} ms  node_batch wall {1e3 * (t2 - t1):.1f} ms  device {dev_ms:.1f} ms",
          flush=True)
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
net.node_batch(plan.path, plan.var, runs, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
