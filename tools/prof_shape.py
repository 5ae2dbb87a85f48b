"""One forced-mode CGEMM of a given shape, a few reps (for ncu captures).

    python tools/prof_shape.py 2048 16384 64 TF32TCEC [variant]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "TF32TCEC"
h = Handle(0)
if len(sys.argv) > 5:
    h.set_gemm_variant(sys.argv[5])
dev = torch.device("cuda:0")
a = (torch.rand(m, k, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
b = (torch.rand(k, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
c = torch.empty(m, n, dtype=torch.complex64, device=dev)
for _ in range(3):
    h.dispatch_cgemm(a, b, make_config(force=mode), out=c)
torch.cuda.synchronize()
