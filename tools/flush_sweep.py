"""Cost of the per-k-block RN flush on the default (wide) kernel: FP16TCEC /
TF32TCEC time at flush interval 1, 2, 4 and 0 (no flush)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
dev = torch.device("cuda:0")
for nn in [int(v) for v in os.environ.get("NS", "4096,8192").split(",")]:
    a = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    b = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    c = torch.empty(nn, nn, dtype=torch.complex64, device=dev)
    for mode in os.environ.get("MODES", "FP16TCEC,TF32TCEC").split(","):
        for fl in (1, 2, 4, 0):
            h.flush_kblocks = fl
            cfg = make_config(force=mode)
            h.dispatch_cgemm(a, b, cfg, out=c)
            h.profile(True)
            for _ in range(5):
                h.dispatch_cgemm(a, b, cfg, out=c)
            st, cnt = h.profile_read()
            h.profile(False)
            g = st["gemm"] / cnt
            print(f"n={nn} {mode} flush={fl}: {g:.3f} ms  {24 * nn**3 / g / 1e9:.0f} TFLOP/s tensor", flush=True)
    h.flush_kblocks = 1
