"""Skinny FP32-tier shapes (k <= 32, one outer dim <= 16): time and HBM floor fraction."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config(force="FP32_REF")
SHAPES = [(2, 1 << 26, 2), (8, 1 << 24, 8), (16, 1 << 22, 16), (16, 1 << 24, 16), (4, 1 << 24, 32),
          (1 << 24, 8, 8), (1 << 26, 2, 2), (1 << 22, 32, 8), (1 << 21, 16, 32), (1 << 20, 16, 16)]
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
for (m, n, k) in SHAPES:
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
