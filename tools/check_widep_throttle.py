"""Bit-identity of the persistent wide kernel (variant 4, with whatever
TCEC_THROTTLE / TCEC_GROUP_M_P the environment sets) against the
one-tile-per-cluster wide kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(5)
for (m, n, k, mode) in [(4096, 4096, 4096, "TF32TCEC"), (2048, 8192, 3000, "FP16TCEC"), (8192, 4096, 1024, "TF32TCEC")]:
    a = torch.randn(m, k, dtype=torch.complex64, device=dev, generator=g)
    b = torch.randn(k, n, dtype=torch.complex64, device=dev, generator=g)
    cfg = make_config(force=mode)
    h.set_gemm_variant("wide")
    c0, _ = h.dispatch_cgemm(a, b, cfg)
    h.set_gemm_variant("wide_persistent")
    c1, _ = h.dispatch_cgemm(a, b, cfg)
    same = torch.equal(c0.view(torch.float32), c1.view(torch.float32))
    print(f"({m},{n},{k}) {mode}: bit-identical {same}", flush=True)
    assert same
