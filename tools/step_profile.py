"""Per-step-shape profile of one Sycamore slice: every distinct (m, n, k) of the
sliced plan dispatched alone (AUTO-0 default policy, random data), time and
throughput, sorted by total time (count x time)."""
import collections
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.paths import _drop_labels  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 12
d = json.load(open(os.path.join(ROOT, "paper_2303_08989_b200", "plans", f"sycamore_m{cyc}.json")))
spec = circuit_to_network(sycamore_like(cyc, 1), [(q * 7 + 3) % 2 for q in range(53)])
sub = _drop_labels(spec, d["sliced"])
live = {i: list(zip(ls, ds)) for i, (ls, ds) in enumerate(zip(sub.labels, sub.dims))}
nxt = len(sub.labels)
shapes = collections.Counter()
for a, b in d["path"]:
    A, B = live.pop(a), live.pop(b)
    la, lb = {l for l, _ in A}, {l for l, _ in B}
    m = math.prod(x for l, x in A if l not in lb)
    n = math.prod(x for l, x in B if l not in la)
    k = math.prod(x for l, x in A if l in lb)
    live[nxt] = [(l, x) for l, x in A if l not in lb] + [(l, x) for l, x in B if l not in la]
    nxt += 1
    if m * n * k >= 1 << 20:
        shapes[(m, n, k)] += 1
h = Handle(0)
dev = torch.device("cuda:0")
cfg = make_config()
rows = []
for (m, n, k), cnt in shapes.items():
    a = torch.randn(m, k, dtype=torch.complex64, device=dev)
    b = torch.randn(k, n, dtype=torch.complex64, device=dev)
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    _, res = h.dispatch_cgemm(a, b, cfg, out=c)
    h.profile(True)
    for _ in range(3):
        h.dispatch_cgemm(a, b, cfg, out=c)
    st, nn = h.profile_read()
    h.profile(False)
    ms = sum(st.values()) / nn
    rows.append((cnt * ms, cnt, (m, n, k), res.line.split(",")[3], ms,
                 8 * m * n * k / ms / 1e9, 8 * (m * k + k * n + m * n) / ms / 1e6))
    del a, b, c
    torch.cuda.empty_cache()
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"total GEMM time per slice (steps >= 2^20 MACs): {tot:.2f} ms")
for r in rows[:int(os.environ.get("TOP", "25"))]:
    print(f"{r[0]:7.2f} ms  x{r[1]:<3d} {str(r[2]):26s} {r[3]:16s} {r[4]:7.3f} ms  {r[5]:7.1f} TF  {r[6]:6.0f} GB/s")
