"""Host overhead of the 4x4 RQC batch call: time per call for 1 vs 65536 bitstrings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402

h = Handle(0)
circ = rqc_rectangular(4, 4, 8, 1)
allx = np.array([[(v >> q) & 1 for q in range(16)] for v in range(1 << 16)], np.uint8)
net = Network(h, circuit_to_network(circ, allx[0]))
path = net.greedy_path()
cfg = make_config()
for n in (1, 1024, 65536):
    xs = allx[:n]
    net.selector_batch(path, xs, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        net.selector_batch(path, xs, cfg)
    dt = (time.perf_counter() - t0) / 10
    print(f"{n} bitstrings: {dt * 1e3:.3f} ms per call", flush=True)
