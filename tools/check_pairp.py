"""Quick check of the persistent 256x128 pair kernel (variant 6) against the
f64 oracle on a few shapes (both formats, both layouts, AUTO/scaled)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2303_08989_b200 import Handle, SelectionPolicy  # noqa: E402
from tests.golden.recipes import matrix_recipe  # noqa: E402

h = Handle(0)
orc = O.oracle()
dev = torch.device("cuda:0")
for (m, n, k) in [(300, 257, 31), (513, 385, 129), (256, 4096, 64), (130, 600, 1100), (2048, 1024, 64), (600, 300, 2100)]:
    a = matrix_recipe("uniform", m, k, 3 + m)
    b = matrix_recipe("uniform", k, n, 5 + n)
    ref = orc.cgemm_oracle(a, b)
    e32 = np.linalg.norm(orc.cgemm(a, b, "FP32_REF")[0].astype(np.complex128) - ref) / np.linalg.norm(ref)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    out = {}
    for var in ("wide", "pair_persistent"):
        h.set_gemm_variant(var)
        for layout in ("a", "b"):
            h.set_operand_layout(layout)
            for mode in ("FP16TCEC", "TF32TCEC"):
                c, _ = h.cgemm(ad, bd, mode)
                cn = c.cpu().numpy()
                err = np.linalg.norm(cn.astype(np.complex128) - ref) / np.linalg.norm(ref)
                out[(var, layout, mode)] = cn
                ok = err <= max(4 * e32, 2e-7)
                print(f"({m},{n},{k}) {var:16s} {layout} {mode}: err {err:.2e} (fp32 {e32:.2e}) {'ok' if ok else 'FAIL'}",
                      flush=True)
            c, res = h.dispatch_cgemm(ad * 2.0 ** -20, bd, SelectionPolicy(size_auto=1, size_tf32=1))
            err = np.linalg.norm(c.cpu().numpy().astype(np.complex128) * 2.0 ** 20 - ref) / np.linalg.norm(ref)
            print(f"   AUTO {res.line.split(',')[3]} err {err:.2e}", flush=True)
    h.set_gemm_variant("auto")
    h.set_operand_layout("auto")
    same = all(np.array_equal(out[("wide", l, md)].view(np.uint32), out[("pair_persistent", l, md)].view(np.uint32))
               for l in ("a", "b") for md in ("FP16TCEC", "TF32TCEC"))
    print("  bit-identical to wide:", same, flush=True)
