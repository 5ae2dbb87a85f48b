import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_2303_08989_b200 import Handle, make_config
h = Handle(0); dev = torch.device('cuda:0')
for n in [int(v) for v in os.environ.get("NS", "1024,2048,4096").split(",")]:
    a = (torch.rand(n, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    b = (torch.rand(n, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    c = torch.empty(n, n, dtype=torch.complex64, device=dev)
    cfg = make_config()
    for _ in range(5): h.dispatch_cgemm(a, b, cfg, out=c)
    torch.cuda.synchronize()
    h.profile(True)
    for _ in range(50): h.dispatch_cgemm(a, b, cfg, out=c)
    st, cnt = h.profile_read(); h.profile(False)
    tot = sum(st.values()) / cnt
    print(n, {k: round(v / cnt * 1e3, 1) for k, v in st.items()}, 'us total', round(tot * 1e3, 1), 'TF', round(8 * n**3 / (tot * 1e-3) / 1e12, 1))
