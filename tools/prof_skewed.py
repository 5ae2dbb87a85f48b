"""configs[2] skewed shapes exactly as bench.py's skewed leg runs them (Type-3
wide-exponent-range operands, size_auto = size_tf32 = min(m, n, k)), a few
AUTO dispatches each -- for an ncu launch list (per-kernel durations).

    ncu --metrics gpu__time_duration.sum --csv python tools/prof_skewed.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, SelectionPolicy, make_config  # noqa: E402

dev = torch.device("cuda:0")
h = Handle(0)
gen = torch.Generator(device=dev)
gen.manual_seed(11)
shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or bench.SKEWED_SHAPES
for (m, n, k) in shapes:
    a, b = bench.type3_device(m, k, gen, dev), bench.type3_device(k, n, gen, dev)
    mn = min(m, n, k)
    cfg = make_config(SelectionPolicy(size_auto=mn, size_tf32=mn))
    c = torch.empty((m, n), dtype=torch.complex64, device=dev)
    for _ in range(3):
        _, res = h.dispatch_cgemm(a, b, cfg, out=c)
    torch.cuda.synchronize()
    print(m, n, k, res.line.split(",")[3], flush=True)
