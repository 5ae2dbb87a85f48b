"""One slice of the Sycamore-class plan (for ncu launch lists / FP32-vs-AUTO fidelity).

    python tools/probe_syc_one.py [cycles] [config: AUTO|FP32_REF]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402
from paper_2303_08989_b200.slicing import SlicePlan, assignment, slice_spec  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 12
mode = sys.argv[2] if len(sys.argv) > 2 else "AUTO"
circ = sycamore_like(cyc, 1)
spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
path, sliced, kind = bench.load_or_build_plan(spec, cyc, "plan")
plan = SlicePlan.build(spec, path, sliced)
h = Handle(0)
net = Network(h, plan.base)
cfg = make_config() if mode == "AUTO" else make_config(force=mode)
vals = net.node_batch(plan.path, plan.var, [plan.run_data(0)], cfg)
torch.cuda.synchronize()
z = complex(vals[0])
if os.environ.get("NOREF"):  # ncu launch lists: one slice only
    sys.exit(0)
ref = bench.contract_f64(h, slice_spec(spec, plan.sliced, assignment(0, plan.dims)), path)
print(kind, mode, "slice0", z, "c128", ref, "rel_err", abs(z - ref) / abs(ref))
import time  # noqa: E402
for nrun in (1, 4):
    runs = [plan.run_data(i) for i in range(nrun)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    net.node_batch(plan.path, plan.var, runs, cfg)
    torch.cuda.synchronize()
    print(f"{nrun} slices: {(time.perf_counter() - t0) * 1e3 / nrun:.1f} ms per slice", flush=True)
