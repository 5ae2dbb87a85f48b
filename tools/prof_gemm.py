"""Profiling driver: a few dispatches of one CGEMM configuration (for ncu).

    python tools/prof_gemm.py --n 4096 --mode AUTO --flush 1 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=4096)
p.add_argument("--m", type=int, default=0)
p.add_argument("--k", type=int, default=0)
p.add_argument("--mode", default="AUTO")
p.add_argument("--flush", type=int, default=-1)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--variant", default="auto")
p.add_argument("--ref-inputs", action="store_true",
               help="configs[1] operands from the reference generator Rng(1 + n) (square only)")
a = p.parse_args()
m, n, k = a.m or a.n, a.n, a.k or a.n
dev = torch.device("cuda:0")
h = Handle(0)
if a.flush >= 0:
    h.flush_kblocks = a.flush
h.set_gemm_variant(a.variant)
if a.ref_inputs:
    from paper_2303_08989_b200.workload import sweep_operands
    Ah, Bh = sweep_operands(n, m=m, k=k)
    A, B = Ah.to(dev), Bh.to(dev)
else:
    A = (torch.rand(m, k, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    B = (torch.rand(k, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
C = torch.empty(m, n, dtype=torch.complex64, device=dev)
cfg = make_config() if a.mode == "AUTO" else make_config(force=a.mode)
for _ in range(a.reps):
    _, res = h.dispatch_cgemm(A, B, cfg, out=C)
torch.cuda.synchronize()
print(res.line)
