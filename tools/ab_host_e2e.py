"""e2e of the host-buffer dispatch (pinned numpy buffers) at given sizes on the
reference inputs: TFLOP/s per call, best of a few (A/B of host-pipeline knobs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.workload import sweep_operands  # noqa: E402

h = Handle(0)
cfg = make_config()
for n in [int(v) for v in sys.argv[1:]] or [8192, 16384]:
    ah, bh = sweep_operands(n)
    a = torch.empty_like(ah).pin_memory().numpy()
    b = torch.empty_like(bh).pin_memory().numpy()
    a[...] = ah.numpy()
    b[...] = bh.numpy()
    c = torch.empty((n, n), dtype=torch.complex64).pin_memory().numpy()
    h.dispatch_cgemm_host(a, b, cfg, out=c)
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        h.dispatch_cgemm_host(a, b, cfg, out=c)
        best = min(best, time.perf_counter() - t0)
    _, res = h.dispatch_cgemm_host(a, b, cfg, out=c)
    print(f"{n}: e2e {8.0 * n ** 3 / best / 1e12:.1f} TFLOP/s ({best * 1e3:.1f} ms) {res.line.split(',')[3]} "
          f"pipeline runs/reruns {h.host_pipeline_stats()}", flush=True)
