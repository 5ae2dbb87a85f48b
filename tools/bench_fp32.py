"""FP32_REF tier throughput (bit-exact SIMT CGEMM) on square and contraction-like shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config(force="FP32_REF")
for (m, n, k) in [(4096, 4096, 4096), (256, 32768, 512), (2048, 131072, 64), (64, 4194304, 64),
                  (8388608, 32, 32), (1024, 16384, 128)]:
    a = torch.randn(m, k, dtype=torch.complex64, device=dev)
    b = torch.randn(k, n, dtype=torch.complex64, device=dev)
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    h.dispatch_cgemm(a, b, cfg, out=c)
    h.profile(True)
    for _ in range(3):
        h.dispatch_cgemm(a, b, cfg, out=c)
    st, cnt = h.profile_read()
    h.profile(False)
    ms = st["gemm"] / cnt
    print(f"({m},{n},{k}): {ms:.3f} ms  {8 * m * n * k / ms / 1e9:.1f} TFLOP/s  "
          f"{8 * (m * k + k * n + m * n) / ms / 1e6:.0f} GB/s", flush=True)
    del a, b, c
