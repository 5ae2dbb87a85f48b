"""AUTO dispatches of the configs[1] sweep sizes on the reference's own inputs
(Rng(1 + n)): whole-dispatch device time (CUDA events) and useful TFLOP/s,
for A/B of tuning knobs given as environment variables.

    python tools/ab_small_auto.py 1024 2048 4096
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.workload import sweep_operands  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config()
for n in [int(v) for v in sys.argv[1:]] or [1024, 2048, 4096]:
    a, b = sweep_operands(n)
    a, b = a.to(dev), b.to(dev)
    c = torch.empty((n, n), dtype=torch.complex64, device=dev)
    for _ in range(3):
        _, res = h.dispatch_cgemm(a, b, cfg, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(torch.cuda.current_stream())
    for _ in range(reps):
        h.dispatch_cgemm(a, b, cfg, out=c)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{n}: {res.line.split(',')[3]} {ms * 1e3:.1f} us  {8.0 * n ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
