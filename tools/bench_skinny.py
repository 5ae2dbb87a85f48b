"""Skinny FP32-tier shapes (k <= 32, one outer dim <= 16): time and HBM floor fraction."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config(force="FP32_REF")
for (m, n, k) in [(2, 1 << 26, 2), (8, 1 << 24, 8), (16, 1 << 22, 16), (16, 1 << 24, 16), (4, 1 << 24, 32),
                  (1 << 24, 8, 8), (1 << 26, 2, 2)]:
    a = torch.randn(m, k, dtype=torch.complex64, device=dev)
    b = torch.randn(k, n, dtype=torch.complex64, device=dev)
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    h.dispatch_cgemm(a, b, cfg, out=c)
    h.profile(True)
    for _ in range(5):
        h.dispatch_cgemm(a, b, cfg, out=c)
    st, cnt = h.profile_read()
    h.profile(False)
    ms = st["gemm"] / cnt
    print(f"({m},{n},{k}): {ms:.3f} ms  {8 * (m * k + k * n + m * n) / ms / 1e6:.0f} GB/s", flush=True)
    del a, b, c
    torch.cuda.empty_cache()
