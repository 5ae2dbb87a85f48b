"""Development probe: deep-circuit amplitudes (configs[4], 7x7 lattice) through
the per-step executor: time per amplitude per mode, accuracy vs the f64 TN
oracle (reference build when present), decision histogram."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2303_08989_b200 import Handle, SelectionPolicy, make_config  # noqa: E402
from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular  # noqa: E402
from paper_2303_08989_b200.network import Network  # noqa: E402
from paper_2303_08989_b200.slicing import contraction_cost  # noqa: E402

h = Handle(0)
ref = O.reference()
depths = [int(d) for d in (sys.argv[1:] or ["12", "16"])]
for depth in depths:
    circ = rqc_rectangular(7, 7, depth, 1)
    xs = bitstrings_for(49, 3, 1)
    spec = circuit_to_network(circ, xs[0])
    t0 = time.perf_counter()
    net = Network(h, spec)
    path = net.greedy_path()
    tp = time.perf_counter() - t0
    big, macs = contraction_cost(spec, path)
    print(f"7x7 d{depth}: {len(path)} steps, max intermediate {big}, {8*macs/1e9:.1f} GFLOP, "
          f"path {tp*1e3:.0f} ms", flush=True)
    tn = None
    if ref is not None and depth <= 12:
        out = (C.c_double * 2)()
        ref.lib.ref_rqc_amplitude_tn_oracle.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                        C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
        ref.lib.ref_rqc_amplitude_tn_oracle(7, 7, depth, 1, (C.c_uint8 * 49)(*xs[0]), out)
        tn = complex(out[0], out[1])
    for label, cfg in (("FP32_REF", make_config(force="FP32_REF")),
                       ("AUTO-0", make_config()),
                       ("AUTO-0-lowered", make_config(SelectionPolicy(size_auto=256, size_tf32=64))),
                       ("TF32TCEC", make_config(force="TF32TCEC")),
                       ("FP16TCEC_SCALED", make_config(force="FP16TCEC_SCALED"))):
        try:
            t, lines = net.contract(path, cfg, want_log=True)
            torch.cuda.synchronize()
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):
                t = net.contract(path, cfg)
            dt = (time.perf_counter() - t0) / reps
            t0 = time.perf_counter()
            amps = net.selector_batch(path, xs, cfg)
            db = (time.perf_counter() - t0) / len(xs)
            hist = {}
            for ln in lines:
                k = ln.split(",")[3]
                hist[k] = hist.get(k, 0) + 1
            err = abs(complex(t.data[0]) - tn) / abs(tn) if tn is not None else float("nan")
            print(f"  {label:16s} contract {dt*1e3:8.2f} ms  graph-batch {db*1e3:8.2f} ms/amp  "
                  f"rel_err_vs_f64 {err:.2e}  |z|={abs(complex(t.data[0])):.3e}  {hist}", flush=True)
        except Exception as e:  # report and continue
            print(f"  {label}: {type(e).__name__}: {e}", flush=True)
    net.close()
