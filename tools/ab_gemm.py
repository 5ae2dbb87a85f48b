"""A/B of tcgen05 kernel variants on square CGEMMs, interleaved, with the SM
clock sampled (NVML) right after each timed batch.

    VARIANTS=wide,wide_np NS=4096,8192 MODES=FP16TCEC python tools/ab_gemm.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2303_08989_b200 import Handle, make_config  # noqa: E402

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
h = Handle(0)
dev = torch.device("cuda:0")
stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
VARIANTS = os.environ.get("VARIANTS", "wide,wide_np").split(",")
NS = [int(x) for x in os.environ.get("NS", "4096,8192").split(",")]
MODES = os.environ.get("MODES", "FP16TCEC").split(",")
ROUNDS = int(os.environ.get("ROUNDS", "2"))
SHAPES = os.environ.get("SHAPES", "")
shapes = [(n, n, n) for n in NS]
if SHAPES:
    shapes = [tuple(int(v) for v in s.split("x")) for s in SHAPES.split(",")]
for (m, n, k) in shapes:
    a = (torch.rand(m, k, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    b = (torch.rand(k, n, 2, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
    c = torch.empty(m, n, dtype=torch.complex64, device=dev)
    reps = max(3, int(2e12 / (8.0 * m * n * k)))
    for rnd in range(ROUNDS):
        for mode in MODES:
            cfg = make_config(force=mode) if mode != "AUTO" else make_config()
            for v in VARIANTS:
                h.set_gemm_variant(v)
                h.dispatch_cgemm(a, b, cfg, out=c)
                h.profile(True)
                torch.cuda.synchronize()
                for _ in range(reps):
                    h.dispatch_cgemm(a, b, cfg, out=c)
                clk = pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)
                pw = pynvml.nvmlDeviceGetPowerUsage(nv) / 1000
                st, cnt = h.profile_read()
                h.profile(False)
                g = st["gemm"] / cnt
                tot = sum(st.values()) / cnt
                fl = 8.0 * m * n * k
                print(f"r{rnd} {m}x{n}x{k} {mode:9s} {v:8s} gemm {g:8.3f} ms {fl / g / 1e9:7.1f} TF "
                      f"(tensor {3 * fl / g / 1e9:6.0f}) step {fl / tot / 1e9:7.1f} TF  sm {clk} MHz {pw:.0f} W",
                      flush=True)
    h.set_gemm_variant("auto")
    del a, b, c
    torch.cuda.empty_cache()
