"""Cost of pinning pageable host memory in place (cudaHostRegister /
cudaHostUnregister) against copying it through a pinned buffer."""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
for gib in (0.5, 2.0):
    n = int(gib * (1 << 30))
    a = np.ones(n, dtype=np.uint8)  # pageable, touched
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, n, 0)
    t1 = time.perf_counter()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    u = cr.cudaHostUnregister(a.ctypes.data)
    t4 = time.perf_counter()
    p = torch.empty(n, dtype=torch.uint8).pin_memory()
    t5 = time.perf_counter()
    np.copyto(p.numpy(), a)
    t6 = time.perf_counter()
    print(f"{gib} GiB: register {t1 - t0:.3f} s ({n / (t1 - t0) / 1e9:.1f} GB/s) rc={r}, H2D from registered "
          f"{n / (t3 - t2) / 1e9:.1f} GB/s, unregister {t4 - t3:.3f} s rc={u}, memcpy into pinned "
          f"{n / (t6 - t5) / 1e9:.1f} GB/s (1 thread)", flush=True)
    del d, p
