"""Permute throughput on rank-r dim-2 tensors (circuit intermediates): GB/s of
16 B per element (read + write) for random permutations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
g = np.random.default_rng(0)
for r in (20, 24, 27):
    t = torch.randn(*([2] * r), dtype=torch.complex64, device=dev)
    for trial in range(3):
        axis = [int(v) for v in g.permutation(r)]
        out = handle_out = h.permute(t, axis)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 10
        for _ in range(reps):
            h.permute(t, axis)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"r={r} perm{trial}: {ms:.3f} ms  {16 * 2**r / ms / 1e6:.0f} GB/s", flush=True)
