"""A/B of the tcgen05 kernel variants on given shapes (forced kind, uniform
operands): GEMM-stage device time (CUDA events) per variant.

    python tools/ab_variant.py TF32TCEC 512,524288,512 512,16384,512 ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

mode = sys.argv[1]
shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[2:]]
variants = os.environ.get("VARIANTS", "wide,wide_persistent,single").split(",")
h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config(force=mode)
for (m, n, k) in shapes:
    a = torch.randn(m, k, dtype=torch.complex64, device=dev)
    b = torch.randn(k, n, dtype=torch.complex64, device=dev)
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    row = []
    for v in variants:
        h.set_gemm_variant(v)
        for _ in range(2):
            h.dispatch_cgemm(a, b, cfg, out=c)
        h.profile(True)
        for _ in range(5):
            h.dispatch_cgemm(a, b, cfg, out=c)
        st, cnt = h.profile_read()
        h.profile(False)
        g = st["gemm"] / cnt
        row.append(f"{v}: {g:.3f} ms ({3 * 8.0 * m * n * k / g / 1e9:.0f} TF/s tensor)")
    h.set_gemm_variant("auto")
    print(f"({m},{n},{k}) {mode}: " + " | ".join(row), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
