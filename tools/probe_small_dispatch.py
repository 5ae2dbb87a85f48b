"""One AUTO dispatch of a small skewed shape (stats -> select -> prep -> GEMM),
a few reps, for ncu launch lists: python tools/probe_small_dispatch.py 256 16384 64"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, SelectionPolicy  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
h = Handle(0)
dev = torch.device("cuda:0")
a = (torch.rand(m, k, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
b = (torch.rand(k, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
c = torch.empty(m, n, dtype=torch.complex64, device=dev)
pol = SelectionPolicy(size_auto=16, size_tf32=8)
for _ in range(4):
    h.dispatch_cgemm(a, b, pol, out=c)
torch.cuda.synchronize()
h.profile(True)
for _ in range(20):
    h.dispatch_cgemm(a, b, pol, out=c)
st, cnt = h.profile_read()
print({k2: round(v / cnt * 1e3, 1) for k2, v in st.items()}, "us")
