"""One slice of the Sycamore-class m=10 plan (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_08989_b200 import Handle, make_config
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like
from paper_2303_08989_b200.network import Network
from paper_2303_08989_b200.paths import random_greedy_path
from paper_2303_08989_b200.slicing import SlicePlan, find_slices
cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 10
circ = sycamore_like(cyc, 1)
spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
path, _, _ = random_greedy_path(spec, trials=64, max_width=30)
plan = SlicePlan.build(spec, path, find_slices(spec, path, n_labels=6))
h = Handle(0)
net = Network(h, plan.base)
vals = net.node_batch(plan.path, plan.var, [plan.run_data(0)], make_config())
torch.cuda.synchronize()
print(vals)
