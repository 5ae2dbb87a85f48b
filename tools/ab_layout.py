"""A/B of the operand layouts (tcec_set_operand_layout: "b" = B-expanded,
"a" = A-expanded, "auto") on the configs[2] skewed shapes and the big
tensor-core steps of the Sycamore m=12 slices: per-stage device time
(statistics / preparation / GEMM, CUDA events) of AUTO dispatches on Type-3
operands (the TF32TCEC fallback), plus the max |difference| between layouts.

    python tools/ab_layout.py [m,n,k ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_08989_b200 import Handle, SelectionPolicy, make_config  # noqa: E402

dev = torch.device("cuda:0")
h = Handle(0)
gen = torch.Generator(device=dev)
gen.manual_seed(11)
shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or (
    bench.SKEWED_SHAPES + [(512, 524288, 512), (4096, 2048, 65536), (65536, 4096, 512)])
reps = int(os.environ.get("REPS", "10"))
for (m, n, k) in shapes:
    a, b = bench.type3_device(m, k, gen, dev), bench.type3_device(k, n, gen, dev)
    mn = min(m, n, k)
    cfg = make_config(SelectionPolicy(size_auto=mn, size_tf32=mn))
    c = torch.empty((m, n), dtype=torch.complex64, device=dev)
    outs, row = {}, []
    for layout in ("b", "a", "auto"):
        h.set_operand_layout(layout)
        for _ in range(3):
            _, res = h.dispatch_cgemm(a, b, cfg, out=c)
        h.profile(True)
        torch.cuda.synchronize()
        for _ in range(reps):
            h.dispatch_cgemm(a, b, cfg, out=c)
        st, cnt = h.profile_read()
        h.profile(False)
        ms = {kk: v / max(cnt, 1) for kk, v in st.items()}
        tot = sum(ms.values())
        tf = 8.0 * m * n * k / (tot * 1e-3) / 1e12
        row.append(f"{layout}: {tot * 1e3:8.1f} us (stats {ms['stats'] * 1e3:6.1f} prep {ms['prep'] * 1e3:7.1f} "
                   f"gemm {ms['gemm'] * 1e3:8.1f}) {tf:6.1f} TF/s")
        outs[layout] = c.clone()
    h.set_operand_layout("auto")
    d = float((outs["a"] - outs["b"]).abs().max()) / max(float(outs["b"].abs().max()), 1e-30)
    print(f"({m},{n},{k}) {res.line.split(',')[3]}  " + " | ".join(row) + f"  max|a-b|/max|b| {d:.2e}",
          flush=True)
    del a, b, c, outs
    torch.cuda.empty_cache()
