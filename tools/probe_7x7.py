"""One 7x7 depth-16 RQC amplitude on the reference's greedy path (AUTO-0), for
ncu launch lists: the per-step kernels of the configs[4] leg."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 16
circ = rqc_rectangular(7, 7, depth, 1)
x = bitstrings_for(49, 10, 1)[0]
spec = circuit_to_network(circ, x)
h = Handle(0)
net = Network(h, spec)
path = net.greedy_path()
cfg = make_config()
net.contract(path, cfg)  # plan + graph capture
torch.cuda.synchronize()
net.contract(path, cfg)
torch.cuda.synchronize()
