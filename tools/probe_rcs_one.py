"""One 7x7 (1+16+1) amplitude through the per-step executor (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_08989_b200 import Handle, make_config
from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular
from paper_2303_08989_b200.network import Network
depth = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = sys.argv[2] if len(sys.argv) > 2 else "AUTO"
h = Handle(0)
circ = rqc_rectangular(7, 7, depth, 1)
net = Network(h, circuit_to_network(circ, bitstrings_for(49, 1, 1)[0]))
path = net.greedy_path()
cfg = make_config() if mode == "AUTO" else make_config(force=mode)
z = net.contract(path, cfg).data[0]
torch.cuda.synchronize()
print(depth, mode, z)
import time  # noqa: E402
from paper_2303_08989_b200.circuits import bitstrings_for as _bs  # noqa: E402
xs = _bs(49, 10, 1)
net.selector_batch(path, xs[:1], cfg)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    net.selector_batch(path, xs, cfg)
    torch.cuda.synchronize()
    print(f"rep {rep}: {(time.perf_counter() - t0) / len(xs) * 1e3:.2f} ms per amplitude", flush=True)
