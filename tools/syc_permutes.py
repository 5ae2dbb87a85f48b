"""The TTGT operand permutes of one Sycamore slice (the sliced plan, label
order as network.cu builds it: A -> free_a|shared, B -> shared|free_b), each
timed alone on the device; prints the slowest with their axis maps.

    python tools/syc_permutes.py [cycles] [top]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle  # noqa: E402
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.paths import _drop_labels  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 12
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
d = json.load(open(os.path.join(ROOT, "paper_2303_08989_b200", "plans", f"sycamore_m{cyc}.json")))
spec = circuit_to_network(sycamore_like(cyc, 1), [(q * 7 + 3) % 2 for q in range(53)])
sub = _drop_labels(spec, d["sliced"])
live = {i: (list(ls), list(ds)) for i, (ls, ds) in enumerate(zip(sub.labels, sub.dims))}
nxt = len(sub.labels)
perms = []
for a, b in d["path"]:
    (la, da), (lb, db) = live.pop(a), live.pop(b)
    shared = [l for l in la if l in lb]
    free_a = [l for l in la if l not in lb]
    free_b = [l for l in lb if l not in la]
    for labels, dims, order in ((la, da, free_a + shared), (lb, db, shared + free_b)):
        axis = [labels.index(l) for l in order]
        if axis != list(range(len(axis))) and math.prod(dims) >= 1 << 16:
            perms.append((dims, axis))
    live[nxt] = (free_a + free_b, [da[la.index(l)] for l in free_a] + [db[lb.index(l)] for l in free_b])
    nxt += 1
h = Handle(0)
dev = torch.device("cuda:0")
rows = []
for dims, axis in perms:
    t = torch.randn(*dims, dtype=torch.complex64, device=dev)
    h.permute(t, axis)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        h.permute(t, axis)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    n = math.prod(dims)
    rows.append((ms, n, 16 * n / ms / 1e6, dims, axis))
    del t
    torch.cuda.empty_cache()
rows.sort(reverse=True)
print(f"{len(rows)} permutes, total {sum(r[0] for r in rows):.2f} ms per slice")
for ms, n, gbs, dims, axis in rows[:top]:
    print(f"{ms:7.3f} ms  2^{int(math.log2(n))}  {gbs:6.0f} GB/s  rank {len(dims)} "
          f"dims {'x'.join(map(str, dims)) if any(x != 2 for x in dims) else '2^' + str(len(dims))}  axis {axis}")
