"""Diagnostic: is the single-CTA TCEC kernel feed-bound (TMA/L2 bytes) or
MMA/smem-operand bound?  Same 12 MMAs per k-block; TCEC_DIAG_HALF_BYTES=1
loads only the hi tiles (numerically meaningless, timing only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_08989_b200 import Handle
h = Handle(0)
dev = torch.device("cuda:0")
for nn in (4096,):
    a = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    b = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    c = torch.empty(nn, nn, dtype=torch.complex64, device=dev)
    for fl in (1, 0):
        h.flush_kblocks = fl
        for mode in ("FP16TCEC", "TF32TCEC", "FP16TC"):
            h.cgemm(a, b, mode, out=c)
            h.profile(True)
            for _ in range(4):
                h.cgemm(a, b, mode, out=c)
            st, cnt = h.profile_read(); h.profile(False)
            g = st["gemm"] / cnt
            nprod = 1 if mode.endswith("TC") else 3
            print(f"n={nn} flush={fl} {mode}: gemm {g:.2f} ms "
                  f"{8*nn**3/(g*1e-3)/1e12:.1f} TF useful, {nprod*8*nn**3/(g*1e-3)/1e12:.0f} TF tensor", flush=True)
