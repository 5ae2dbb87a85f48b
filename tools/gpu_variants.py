"""Development probe: TCEC kernel variants (single CTA vs CTA pair) x flush
interval: accuracy against the f64 oracle and throughput."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2303_08989_b200 import Handle  # noqa: E402
from tests.golden.recipes import matrix_recipe  # noqa: E402

h = Handle(0)
VARIANTS = os.environ.get("VARIANTS", "single,wide").split(",")
FLUSHES = [int(x) for x in os.environ.get("FLUSHES", "1,0").split(",")]
o = O.oracle()
dev = torch.device("cuda:0")


def relerr(c, ref):
    return float(np.linalg.norm(np.asarray(c, np.complex128) - ref) / np.linalg.norm(ref))


cases = [("uniform", 300, 257, 1000), ("banded", 96, 80, 88), ("uniform", 130, 130, 1100),
         ("uniform", 513, 385, 129)]
for rec, m, n, k in cases:
    a = matrix_recipe(rec, m, k, 3)
    b = matrix_recipe(rec, k, n, 4)
    ref = o.cgemm_oracle(a, b)
    e32 = relerr(o.cgemm(a, b, "FP32_REF")[0], ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    for pair in ("single", "pair", "wide"):
        h.set_gemm_variant(pair)
        for fl in (1, 2, 4):
            h.flush_kblocks = fl
            row = []
            for mode in ("FP16TCEC", "TF32TCEC", "FP16TC"):
                c, _ = h.cgemm(ad, bd, mode)
                row.append(f"{mode}={relerr(c.cpu().numpy(), ref):.2e}")
            print(f"acc {rec} {m}x{n}x{k} pair={pair} flush={fl} fp32ref={e32:.2e} " + " ".join(row),
                  flush=True)

for nn in (4096, 8192):
    a = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    b = (torch.rand(nn, nn, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    c = torch.empty(nn, nn, dtype=torch.complex64, device=dev)
    for pair in VARIANTS:
        h.set_gemm_variant(pair)
        for fl in FLUSHES:
            h.flush_kblocks = fl
            for mode in ("FP16TCEC", "TF32TCEC"):
                h.cgemm(a, b, mode, out=c)
                h.profile(True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                reps = 5
                for _ in range(reps):
                    h.cgemm(a, b, mode, out=c)
                torch.cuda.synchronize()
                dt = (time.perf_counter() - t0) / reps
                st, cnt = h.profile_read()
                h.profile(False)
                g = st["gemm"] / max(cnt, 1)
                print(f"perf n={nn} pair={pair} flush={fl} {mode}: step {dt*1e3:.2f} ms "
                      f"({8*nn**3/dt/1e12:.1f} TF/s)  gemm {g:.2f} ms ({8*nn**3/(g*1e-3)/1e12:.1f} TF/s useful, "
                      f"{24*nn**3/(g*1e-3)/1e12:.0f} tensor)", flush=True)
