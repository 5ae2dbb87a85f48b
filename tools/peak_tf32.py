"""Measured dense TF32 / BF16 tensor peaks on this box (the roofline
denominators of the TF32TCEC path), by the same recipe the driver uses for
MEASURED_PEAKS.json: torch.matmul (cuBLAS) at 8192^3, best of 10 (burst) and
back to back for 4 s (sustained), CUDA events; plus the SM clock under load.

    python tools/peak_tf32.py > profiles/r02_tf32_peak.json
"""
import json
import subprocess
import threading
import time

import torch


def sample_clocks(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "200", "-i", "0"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if not ln:
            break
        try:
            out.append([float(x) for x in ln.split(",")])
        except ValueError:
            pass
    p.terminate()


def measure(dtype, tf32, n=8192, sustain_s=4.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    flops = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    stop, clk = threading.Event(), []
    th = threading.Thread(target=sample_clocks, args=(stop, clk), daemon=True)
    th.start()
    reps = 0
    t0 = time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < sustain_s:
        for _ in range(8):
            torch.matmul(a, b, out=c)
        reps += 8
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    stop.set()
    th.join(timeout=5)
    sust = flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    load = [c[0] for c in clk if c[0] > 500]
    return {"burst_tflops": round(best, 1), "sustained_tflops": round(sust, 1),
            "sm_mhz_median": sorted(load)[len(load) // 2] if load else None,
            "power_w_max": max((c[1] for c in clk), default=None)}


if __name__ == "__main__":
    out = {"gpu": torch.cuda.get_device_name(0),
           "how": "torch.matmul (cuBLAS) 8192^3 (2 N^3 flops): best of 10 = burst, back to back 4 s = "
                  "sustained; fp32 inputs with allow_tf32 for TF32",
           "tf32": measure(torch.float32, True), "bf16": measure(torch.bfloat16, False)}
    print(json.dumps(out))
