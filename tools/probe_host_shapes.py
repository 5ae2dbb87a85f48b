"""Host-buffer dispatch (pinned) on non-square shapes, uniform(-1,1) operands:
e2e TFLOP/s, device-buffer time of the same dispatch, speculation reruns."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

h = Handle(0)
cfg = make_config()
g = np.random.default_rng(3)
for (m, n, k) in [(16384, 4096, 8192), (8192, 16384, 4096), (32768, 2048, 2048), (12288, 12288, 2048),
                  (16384, 16384, 1024), (9000, 7000, 5000)]:
    a = torch.empty((m, k), dtype=torch.complex64).pin_memory().numpy()
    b = torch.empty((k, n), dtype=torch.complex64).pin_memory().numpy()
    a.view(np.float32)[...] = g.random((m, 2 * k), dtype=np.float32) * 2 - 1
    b.view(np.float32)[...] = g.random((k, 2 * n), dtype=np.float32) * 2 - 1
    c = torch.empty((m, n), dtype=torch.complex64).pin_memory().numpy()
    r0 = h.host_pipeline_stats()
    h.dispatch_cgemm_host(a, b, cfg, out=c)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        _, res = h.dispatch_cgemm_host(a, b, cfg, out=c)
        best = min(best, time.perf_counter() - t0)
    r1 = h.host_pipeline_stats()
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    cd = torch.empty((m, n), dtype=torch.complex64, device="cuda")
    h.dispatch_cgemm(ad, bd, cfg, out=cd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        h.dispatch_cgemm(ad, bd, cfg, out=cd)
    dev_s = (time.perf_counter() - t0) / 3
    fl = 8.0 * m * n * k
    print(f"({m},{n},{k}) {res.line.split(',')[3]}: e2e {fl / best / 1e12:.1f} TFLOP/s, device {fl / dev_s / 1e12:.1f}, "
          f"ratio {dev_s / best:.3f}, runs/reruns +{r1[0] - r0[0]}/+{r1[1] - r0[1]}", flush=True)
    del ad, bd, cd
    torch.cuda.empty_cache()
