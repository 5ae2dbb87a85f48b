"""A/B of wide-kernel variants and the TF32 flush interval on the headline
configuration (configs[1] 16384^3 on the reference inputs -> TF32TCEC), plus
the forced FP16TCEC path: device ms per dispatch (CUDA events), K3 share, and
the row-sampled error vs complex128 next to the bit-exact FP32 tier's.

    python tools/ab_headline.py [n] [variants] [flushes] [modes]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.workload import sweep_operands  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
variants = (sys.argv[2] if len(sys.argv) > 2 else "wide,wide_mc").split(",")
flushes = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1").split(",")]
modes = (sys.argv[4] if len(sys.argv) > 4 else "AUTO,FP16TCEC").split(",")
dev = torch.device("cuda:0")
h = Handle(0)
stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
ah, bh = sweep_operands(n)
a, b = ah.to(dev), bh.to(dev)
c = torch.empty(n, n, dtype=torch.complex64, device=dev)
rows = torch.from_numpy(np.random.default_rng(3).choice(n, 8, replace=False)).to(dev)
ref = a[rows].to(torch.complex128) @ b.to(torch.complex128)
c32, _ = h.cgemm(a[rows].contiguous(), b, "FP32_REF")
e32 = float(torch.linalg.norm(c32.to(torch.complex128) - ref) / torch.linalg.norm(ref))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in modes:
    cfg = make_config() if mode == "AUTO" else make_config(force=mode)
    for fl in flushes:
        for v in variants:
            h.set_gemm_variant(v)
            h.flush_kblocks = fl
            for _ in range(2):
                _, res = h.dispatch_cgemm(a, b, cfg, out=c)
            torch.cuda.synchronize()
            h.profile(True)
            e0.record(stream)
            reps = 5
            for _ in range(reps):
                h.dispatch_cgemm(a, b, cfg, out=c)
            e1.record(stream)
            e1.synchronize()
            st, cnt = h.profile_read()
            h.profile(False)
            ms = e0.elapsed_time(e1) / reps
            err = float(torch.linalg.norm(c[rows].to(torch.complex128) - ref) / torch.linalg.norm(ref))
            print(f"{mode:9s} {res.line.split(',')[3]:16s} variant={v:9s} flush={fl} ms={ms:8.3f} "
                  f"TFLOP/s={8.0 * n ** 3 / ms / 1e9:7.1f} gemm_ms={st['gemm'] / cnt:8.3f} "
                  f"err={err:.3e} (fp32 {e32:.3e}, x{err / e32:.2f})", flush=True)
h.set_gemm_variant("auto")
h.flush_kblocks = 1
