"""One skinny FP32-tier contraction step whose long operand needs a TTGT
permute (scattered shared axes), timed through the network executor: with the
fused gather (TCEC_VIEW_GATHER=1, default) or permute + GEMM (=0).

    python tools/bench_skinny_view.py [log2_long] [n_shared] [n_new] [t_first]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import NetworkSpec  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 26
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 6
nn = int(sys.argv[3]) if len(sys.argv) > 3 else 4
t_first = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
g = np.random.default_rng(3)
tl = [f"t{i}" for i in range(L)]
shared = [tl[i] for i in sorted(g.choice(L, ns, replace=False), key=lambda _: g.random())]
gl = shared + [f"n{j}" for j in range(nn)]
rng = np.random.default_rng(1)
data_t = (rng.standard_normal(2 ** L) + 1j * rng.standard_normal(2 ** L)).astype(np.complex64)
data_g = (rng.standard_normal(2 ** len(gl)) + 1j * rng.standard_normal(2 ** len(gl))).astype(np.complex64)
spec = NetworkSpec(labels=[tl, gl], dims=[[2] * L, [2] * len(gl)], data=[data_t, data_g])
h = Handle(0)
net = Network(h, spec)
path = [(0, 1)] if t_first else [(1, 0)]
cfg = make_config()
_, lines = net.contract(path, cfg, want_log=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
s = torch.cuda.ExternalStream(h.stream_ptr) if h.stream_ptr else torch.cuda.current_stream()
e0.record(s)
for _ in range(reps):
    net.contract(path, cfg)
e1.record(s)
torch.cuda.synchronize()
print(f"{lines[0]}  view={os.environ.get('TCEC_VIEW_GATHER', '1')}  {e0.elapsed_time(e1) / reps:.3f} ms per contraction "
      f"(incl. result copy)", flush=True)
