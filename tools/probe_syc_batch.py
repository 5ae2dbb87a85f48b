"""Per-slice cost of node_batch calls of 1 / 4 / 8 / 32 slices on one GPU
(the shares one rank gets at N = 32 / 8 / 4 / 1 GPUs): wall and device time,
to check that the sliced RCS has no per-call overhead that would cap scaling."""
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
net.node_batch(plan.path, plan.var, [plan.run_data(0)], cfg)
for nb in (1, 4, 8, 32):
    ids = list(range(nb))
    net.node_batch(plan.path, plan.var, [plan.run_data(i) for i in ids], cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.profile(True)
    runs = [plan.run_data(i) for i in ids]
    net.node_batch(plan.path, plan.var, runs, cfg)
    t1 = time.perf_counter()
    dev_ms, _ = h.profile_read_batches()
    h.profile(False)
    print(f"{nb:2d} slices: wall {1e3 * (t1 - t0):8.1f} ms ({1e3 * (t1 - t0) / nb:.2f} per slice)  "
          f"device {dev_ms:8.1f} ms ({dev_ms / nb:.2f} per slice)", flush=True)
