#!/usr/bin/env python
"""bench.py -- TCEC CGEMM TFLOP/s (+ fidelity) on B200, BASELINE.json configs[1].

Workload (one "step"): one AUTO-0 dispatch_cgemm (precsel.cpp:225-322 semantics:
device exponent statistics -> selection -> scale+split -> tcgen05 TCEC CGEMM ->
descale) of the top of the configs[1] sweep, m = n = k = 16384, uniform(-1,1)
complex64 inputs (synthetic; the selector picks FP16TCEC_SCALED, s = 15).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value   = useful 8mnk flops / device time (CUDA events on the handle stream), inputs
          resident in HBM; N>1 runs N independent replicas (replicas only: the
          standalone CGEMM does not shard) -> whole-job flops / max time.
e2e     = the same through the host-buffer C-ABI entry point tcec_dispatch_cgemm_host
          (H2D of A and B from pinned memory + dispatch + D2H of C inside the timed region).
roofline= the dominant kernel (tcec_gemm_kernel<f16>), tensor-pipe flops 3 x 8mnk per
          launch over its CUDA-event duration, against the measured dense bf16/fp16 peak.
cpu_baseline / --impl reference = the reference's own kernels (oracle/_ref, the
          unmodified mpsgemm sources) row-partitioned over all host threads on a bounded
          row block of the same CGEMM.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 16384
METRIC = "TCEC CGEMM TFLOP/s (useful 8mnk, AUTO-selected, m=n=k=16384)"
PAPER_A100_FP16TCEC = 54.2  # BASELINE.md / PAPER.md:246, max measured FP16TCEC CGEMM on A100


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------- CPU reference
def cpu_reference_sample(a_host, b_host, budget_s=10.0, threads=None, min_rows=None):
    """The reference's own kernels on a row block of the same CGEMM, all host
    threads (row partitioning is allowed by kernels.hpp:16-19 and bit-identical).
    Returns (tflops, rows, seconds, threads, kind)."""
    import oracle as O
    threads = threads or os.cpu_count() or 1
    n = b_host.shape[1]
    k = b_host.shape[0]
    ref = O.reference()
    m = a_host.shape[0]
    if ref is not None:
        lib = ref.lib
        fn = lib.ref_cgemm_rows_threaded_timed
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                       C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        kind = "reference"

        def run(rows):
            c = np.empty((rows, n), np.complex64)
            prep, gemm = C.c_double(0), C.c_double(0)
            fn(a_host.ctypes.data, b_host.ctypes.data, c.ctypes.data, m, n, k, 0, rows,
               5, 16, threads, C.byref(prep), C.byref(gemm))  # GemmMode::fp16_tcec, k_tile 16
            return prep.value, gemm.value
    else:
        o = O.oracle()
        kind = "port"
        threads = 1

        def run(rows):
            t0 = time.perf_counter()
            o.cgemm(a_host[:rows], b_host, "FP16TCEC")
            return 0.0, time.perf_counter() - t0
    if min_rows is None:
        _, g1 = run(max(1, threads))
        per_row = g1 / max(1, threads)
        rows = int(max(threads, min(m, budget_s / max(per_row, 1e-9))))
        rows = max(threads, (rows // threads) * threads)
    else:
        rows = min_rows
    prep, gemm = run(rows)
    # the full CGEMM runs the O(n^2) preparation once and the row loop m/rows times
    full_s = prep + gemm * m / rows
    return 8.0 * m * n * k / full_s / 1e12, rows, prep + gemm, threads, kind, prep, gemm


# ---------------------------------------------------------------- helpers
def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def host_inputs(n, seed):
    import torch
    g = np.random.default_rng(seed)
    pin = torch.cuda.is_available()
    a = torch.empty((n, n), dtype=torch.complex64, pin_memory=pin)
    b = torch.empty((n, n), dtype=torch.complex64, pin_memory=pin)
    for t in (a, b):
        v = t.numpy().view(np.float32)
        for r0 in range(0, n, 1024):
            v[r0:r0 + 1024] = g.random((min(1024, n - r0), 2 * n), dtype=np.float32) * 2 - 1
    return a, b


# ------------------------------------------------------------------- arms
def run_ours(args):
    import torch
    from paper_2303_08989_b200 import Handle, make_config
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.n
    h = Handle(local)
    stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
    a_h, b_h = host_inputs(n, 1 + n + rank)
    a = a_h.to(dev)
    b = b_h.to(dev)
    c = torch.empty((n, n), dtype=torch.complex64, device=dev)
    cfg = make_config()  # AUTO-0, default SelectionPolicy (size_auto 2048 <= n)
    flops = 8.0 * n * n * n

    for _ in range(args.warmup):
        _, res = h.dispatch_cgemm(a, b, cfg, out=c)
    decision = res.line
    kind = res.line.split(",")[3]

    # ---- device-resident timed region
    h.profile(True)
    barrier(world)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            h.dispatch_cgemm(a, b, cfg, out=c)
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.steps
    stage, cnt = h.profile_read()
    h.profile(False)
    ms_max = max_over_ranks(ms, world)
    gemm_ms = stage["gemm"] / max(cnt, 1)

    # ---- end to end through the host-buffer C-ABI
    a_np, b_np = a_h.numpy(), b_h.numpy()
    c_h = torch.empty((n, n), dtype=torch.complex64, pin_memory=True)
    c_np = c_h.numpy()
    h.dispatch_cgemm_host(a_np, b_np, cfg, out=c_np)  # allocate staging once
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        h.dispatch_cgemm_host(a_np, b_np, cfg, out=c_np)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / args.steps
    e2e_ms = max_over_ranks(e2e_ms, world)
    pipe_runs, pipe_reruns = h.host_pipeline_stats()

    # ---- fidelity: sampled rows vs complex128, and the bit-exact FP32 tier on the same rows
    rows = torch.from_numpy(np.random.default_rng(3).choice(n, 16, replace=False)).to(dev)
    ref = a[rows].to(torch.complex128) @ b.to(torch.complex128)
    err = float(torch.linalg.norm(c[rows].to(torch.complex128) - ref) / torch.linalg.norm(ref))
    c32, _ = h.cgemm(a[rows].contiguous(), b, "FP32_REF")
    err32 = float(torch.linalg.norm(c32.to(torch.complex128) - ref) / torch.linalg.norm(ref))
    del ref

    # ---- small sweep (configs[1] 1024..8192), AUTO and forced formats
    sweep = {}
    if args.sweep and rank == 0:
        for sn in (1024, 2048, 4096, 8192):
            sa = torch.rand(sn, sn, 2, device=dev).mul_(2).sub_(1).view(torch.complex64)[..., 0].contiguous()
            sb = torch.rand(sn, sn, 2, device=dev).mul_(2).sub_(1).view(torch.complex64)[..., 0].contiguous()
            sc = torch.empty(sn, sn, dtype=torch.complex64, device=dev)
            row = {}
            for label, sc_cfg in (("AUTO-0", make_config()), ("FP16TCEC", make_config(force="FP16TCEC")),
                                  ("TF32TCEC", make_config(force="TF32TCEC")),
                                  ("FP32_REF", make_config(force="FP32_REF"))):
                reps = 2 if label == "FP32_REF" else 5
                for _ in range(2):
                    _, r = h.dispatch_cgemm(sa, sb, sc_cfg, out=sc)
                torch.cuda.synchronize(dev)
                e0.record(stream)
                for _ in range(reps):
                    h.dispatch_cgemm(sa, sb, sc_cfg, out=sc)
                e1.record(stream)
                e1.synchronize()
                row[label] = round(8.0 * sn ** 3 / (e0.elapsed_time(e1) / reps * 1e-3) / 1e12, 2)
                if label == "AUTO-0":
                    row["AUTO-0 mode"] = r.line.split(",")[3]
            sweep[str(sn)] = row
            del sa, sb, sc

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        tf, r_rows, dt, thr, kindc, prep, gemm = cpu_reference_sample(a_np, b_np,
                                                                     budget_s=args.cpu_budget)
        cpu = {"value": round(tf, 6), "unit": "TFLOP/s", "cores": thr, "kind": kindc,
               "sample": f"rows 0..{r_rows} of the same m=n=k={n} CGEMM with the reference's "
                         f"FP16TCEC kernels on {thr} threads: operand prep {prep:.1f} s + row "
                         f"GEMM {gemm:.1f} s, extrapolated to all {n} rows (prep once)"}

    if rank == 0:
        bpk, bps, hbm, src = peaks()
        tensor_flops = 3.0 * flops  # hi*hi, lo*hi, hi*lo tensor-core products per launch
        achieved = tensor_flops / (gemm_ms * 1e-3) / 1e12
        peak = bps if kind != "TF32TCEC" else bps / 2
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"tcec_gemm_f16_n{n}")
        value = world * flops / (ms_max * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(value / PAPER_A100_FP16TCEC, 2),
            "baseline_ref": "54.2 TFLOP/s FP16TCEC CGEMM max on A100 (PAPER.md:246)",
            "dtype": "c64 (FP32 via error-corrected FP16 tensor cores)",
            "data": "synthetic uniform(-1,1) complex64 (numpy default_rng), resident in HBM",
            "config": {"workload": f"configs[1] CGEMM sweep top: m=n=k={n}, AUTO-0 "
                                   f"(default SelectionPolicy) -> {kind}",
                       "decision": decision, "parallelism": f"replicas x{world}",
                       "l2": "inputs (2 GiB per operand) exceed the 126 MB L2",
                       "flush_kblocks": h.flush_kblocks},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": gemm_kernel_name(n, n, kind),
                         "note": f"3 x 8mnk tensor-pipe flops per launch / CUDA-event time; "
                                 f"peak = {src} dense bf16 sustained (fp16 = bf16 rate)"},
            "stages_ms": {k2: round(v / max(cnt, 1), 3) for k2, v in stage.items()},
            "fidelity": {"rel_err": err, "fp32_ref_rel_err": err32,
                         "ratio_vs_fp32": round(err / err32, 3) if err32 else None,
                         "sample": "16 random rows vs complex128"},
            "e2e": {"value": round(world * flops / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                    "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * n * 8,
                    "pipeline": {"runs": pipe_runs, "reruns": pipe_reruns,
                                 "note": "H2D of B column parts / A row chunks overlapped with the GEMM "
                                         "blocks under a decision from the first parts, checked against "
                                         "the exact one (reruns = recomputed on disagreement)"}},
            # per AUTO dispatch: stats1, stats2, select, prep_a, prep_b and ONE
            # tcgen05 GEMM (the wide kernel branches on the device decision),
            # plus a cudaMemsetAsync of the decision slot
            "gpu_launches": 6 * args.steps,
            "clocks": clk.summary(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if sweep:
            line["sweep_tflops"] = sweep
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch  # noqa: F401  (pinned inputs share the generator with our arm)
    n = args.n
    a_h, b_h = host_inputs(n, 1 + n)
    a_np, b_np = a_h.numpy(), b_h.numpy()
    # calibrate the bounded per-step sample once, then warm up and time
    _, rows, _, thr, kind, _, _ = cpu_reference_sample(a_np, b_np, budget_s=args.ref_step_s)
    for _ in range(args.warmup):
        cpu_reference_sample(a_np, b_np, min_rows=rows)
    vals, wall = [], 0.0
    for _ in range(args.steps):
        tf, _, dt, _, _, _, _ = cpu_reference_sample(a_np, b_np, min_rows=rows)
        vals.append(tf)
        wall += dt
    value = float(np.mean(vals))
    ms = 8.0 * n * n * n / (value * 1e12) * 1e3  # full-CGEMM time implied by the sample
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c64 (FP32 via error-corrected FP16 emulation, reference CPU)",
        "data": "synthetic uniform(-1,1) complex64",
        "config": {"workload": f"configs[1] CGEMM sweep top: m=n=k={n}, AUTO-0 -> FP16TCEC_SCALED",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": thr, "kind": kind,
                         "sample": f"{rows} rows of the m=n=k={n} CGEMM per step (FP16TCEC "
                                   f"kernels of the unmodified reference, row-partitioned over "
                                   f"{thr} threads; O(n^2) operand prep timed per step and "
                                   f"amortized over the full {n} rows); {wall / args.steps:.1f} s "
                                   f"wall per step"},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


RQC_METRIC = "RCS 4x4 (1+8+1) amplitudes/s (all 2^16 bitstrings, AUTO-0 default policy)"


def rqc_reference_rate(bits, nq, rows, cols, depth, seed, threads, cfg_kw=None):
    """The reference's run_rqc inner loop (one greedy path, contract_network per
    bitstring) over host threads; returns (amplitudes/s, seconds, amplitudes)."""
    import oracle as O
    ref = O.reference()
    if ref is None:
        return None
    fn = ref.lib.ref_rqc_amplitudes_batch
    fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int,
                   C.POINTER(O.ConfigPod), C.c_void_p, C.c_int]
    cfg = O.make_config(**(cfg_kw or {}))
    out = np.empty(len(bits) * 2, np.float32)
    t0 = time.perf_counter()
    rc = fn(rows, cols, depth, seed, bits.ctypes.data, len(bits), C.byref(cfg), out.ctypes.data,
            threads)
    dt = time.perf_counter() - t0
    assert rc == 0
    return len(bits) / dt, dt, out.view(np.complex64)


def statevector_c128(circuit, dev):
    """complex128 state vector of a circuit on the GPU (torch; qubit q = bit q
    of the index): the fidelity reference of the 4x4 leg (the oracle package is
    test infrastructure and stays out of the measured legs)."""
    import torch
    from paper_2303_08989_b200.circuits import CZ, gate_matrix
    n = circuit.n_qubits
    st = torch.zeros(1 << n, dtype=torch.complex128, device=dev)
    st[0] = 1.0
    for layer in circuit.layers:
        for g in layer:
            if g.kind == CZ:
                # index bit q is tensor axis n-1-q of a (2,)*n view
                v = st.view((2,) * n)
                ax_a, ax_b = n - 1 - g.qubits[0], n - 1 - g.qubits[1]
                idx = [slice(None)] * n
                idx[ax_a] = 1
                idx[ax_b] = 1
                v[tuple(idx)] *= -1
                continue
            u = torch.tensor(np.asarray(gate_matrix(g.kind), np.complex128), device=dev)
            if len(g.qubits) == 2:
                u = u.reshape(2, 2, 2, 2)  # (out_a, out_b, in_a, in_b)
                v = st.view((2,) * n)
                ax_a, ax_b = n - 1 - g.qubits[0], n - 1 - g.qubits[1]
                v = torch.tensordot(u, v, dims=([2, 3], [ax_a, ax_b]))  # new axes 0,1 = a, b
                rest = [i for i in range(n) if i not in (ax_a, ax_b)]
                order = [0] * n
                order[ax_a], order[ax_b] = 0, 1
                for pos, ax in enumerate(rest):
                    order[ax] = 2 + pos
                st = v.permute(*order).contiguous().reshape(-1)
            else:
                u = u.reshape(2, 2)
                v = st.view((2,) * n)
                ax = n - 1 - g.qubits[0]
                v = torch.movedim(torch.tensordot(u, v, dims=([1], [ax])), 0, ax)
                st = v.contiguous().reshape(-1)
    return st


def run_rqc(args):
    """configs[0]: 4x4 rectangular RQC, H + 8 CZ layers + H, every output amplitude."""
    import torch
    from paper_2303_08989_b200 import Handle, make_config
    from paper_2303_08989_b200.circuits import circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.network import Network
    rows, cols, depth, seed = 4, 4, 8, 1
    nq = rows * cols
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    circ = rqc_rectangular(rows, cols, depth, seed)
    allx = np.array([[(v >> q) & 1 for q in range(nq)] for v in range(1 << nq)], np.uint8)
    mine = allx[rank::world]
    if args.impl != "reference":
        # the step's host buffers in pinned memory (as the cgemm leg's e2e)
        pin_bits = torch.empty(mine.shape, dtype=torch.uint8, pin_memory=True).numpy()
        pin_bits[...] = mine
        mine = pin_bits
        pin_out = torch.empty(len(mine), dtype=torch.complex64, pin_memory=True).numpy()
    if args.impl == "reference":
        if rank != 0:
            return
        thr = os.cpu_count() or 1
        sample = allx[: min(len(allx), 4096 * max(1, thr // 4))]
        rqc_reference_rate(sample[: 2 * thr], nq, rows, cols, depth, seed, thr)  # warm
        rates = [rqc_reference_rate(sample, nq, rows, cols, depth, seed, thr)[0]
                 for _ in range(max(1, args.steps))]
        value = float(np.mean(rates))
        print(json.dumps({
            "impl": "reference", "metric": RQC_METRIC, "value": round(value, 1),
            "unit": "amplitudes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(len(allx) / value * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c64", "data": "synthetic circuit",
            "config": {"workload": "configs[0] 4x4 RQC (1+8+1), seed 1, all 65536 bitstrings",
                       "parallelism": "host threads"},
            "cpu_baseline": {"value": round(value, 1), "unit": "amplitudes/s", "cores": thr,
                             "kind": "reference",
                             "sample": f"{len(sample)} bitstrings per step, run_rqc loop "
                                       f"(experiments.cpp:211-230) on {thr} threads"},
            "e2e": {"value": round(value, 1), "unit": "amplitudes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    h = Handle(local)
    stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
    net = Network(h, circuit_to_network(circ, [0] * nq))
    path = net.greedy_path()
    cfg = make_config()
    for _ in range(args.warmup):
        amps = net.selector_batch(path, mine, cfg)
    barrier(world)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h.profile(True)  # device time between each batch's uploads and its download
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            amps = net.selector_batch(path, mine, cfg, out=pin_out)
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - t0) / args.steps * 1e3
    dev_ms, n_batches = h.profile_read_batches()
    h.profile(False)
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1) / args.steps, wall), world)
    ms = max_over_ranks(dev_ms / max(n_batches, 1), world)  # bitstrings resident in HBM
    if rank == 0:
        sv = statevector_c128(circ, dev).cpu().numpy()
        idx = np.array([sum(int(b) << q for q, b in enumerate(x)) for x in mine])
        ref = sv[idx]
        err = float(np.max(np.abs(amps.astype(np.complex128) - ref) / np.abs(ref)))
        med = float(np.median(np.abs(amps.astype(np.complex128) - ref) / np.abs(ref)))
        norm = float(np.sum(np.abs(amps.astype(np.complex128)) ** 2)) if world == 1 else None
        cpu = None
        if world == 1 and not args.no_cpu:
            thr = os.cpu_count() or 1
            r = rqc_reference_rate(allx[:4096], nq, rows, cols, depth, seed, thr)
            if r is not None:
                rate, dt, zr = r
                same = bool(np.array_equal(zr.view(np.uint32), amps[:4096].view(np.uint32)))
                cpu = {"value": round(rate, 1), "unit": "amplitudes/s", "cores": thr,
                       "kind": "reference", "bit_identical_to_gpu": same,
                       "sample": f"4096 bitstrings, run_rqc loop on {thr} threads, {dt:.2f} s"}
        value = len(allx) / (ms * 1e-3)
        line = {
            "metric": RQC_METRIC, "value": round(value, 1), "unit": "amplitudes/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64 (FP32 tier, bit-identical to the reference)",
            "data": "synthetic circuit rqc_rectangular(4,4,8,1)",
            "config": {"workload": "configs[0] 4x4 RQC (1+8+1) single-amplitude TTGT contraction, "
                                   "all 65536 bitstrings per step",
                       "executor": "fused small-step kernel (one warp per bitstring)",
                       "steps_per_amplitude": len(path), "parallelism": f"bitstrings / {world}"},
            "fidelity": {"max_rel_err_vs_statevector": err, "median_rel_err": med,
                         "sum_prob": norm},
            "e2e": {"value": round(len(allx) / (e2e_ms * 1e-3), 1), "unit": "amplitudes/s",
                    "ms_per_step": round(e2e_ms, 4),
                    "h2d_bytes_per_step": int(mine.size), "d2h_bytes_per_step": int(len(mine) * 8),
                    "note": "the whole tcec_contract_selector_batch call from host bitstrings to host "
                            "amplitudes; value = its device time after the upload"},
            "gpu_launches": args.steps, "clocks": clk.summary(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    net.close()
    h.close()


SYC_METRIC = "Sycamore-class 53q sliced RCS amplitudes/s (AUTO-0)"


def load_or_build_plan(spec, cycles, mode, log=None):
    """Sliced contraction plan: the committed plans/sycamore_m{cycles}.json
    (made by tools/make_plan.py) when it matches this network, else a fresh
    hyper_path search (mode "hyper") or the randomized greedy (mode "greedy")."""
    from paper_2303_08989_b200.paths import hyper_path, random_greedy_path
    from paper_2303_08989_b200.slicing import find_slices
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from make_plan import spec_hash
    fn = os.environ.get("TCEC_PLAN_FILE") or os.path.join(ROOT, "paper_2303_08989_b200", "plans",
                                                          f"sycamore_m{cycles}.json")
    if mode == "plan" and os.path.exists(fn):
        d = json.load(open(fn))
        if d["spec_hash"] == spec_hash(spec):
            return [tuple(x) for x in d["path"]], list(d["sliced"]), f"hyper (cached {os.path.basename(fn)})"
    if mode == "greedy":
        path, _, _ = random_greedy_path(spec, trials=64, max_width=30)
        return path, find_slices(spec, path, n_labels=6), "randomized greedy"
    path, sliced, _, _ = hyper_path(spec, 28.0, trials=1, log=log)
    return path, sliced, "hyper (searched)"


def run_sycamore(args):
    """configs[3]: 53-qubit Sycamore-layout fSim circuit (m cycles), sliced
    contraction plan (presimplify + partition tree + reconfiguration + exact
    slicing, paths.hyper_path), slices sharded round-robin over the ranks, one
    NCCL all_gather of the slice values, slice-ordered float64 sum."""
    import torch
    from paper_2303_08989_b200 import Handle, make_config
    from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like
    from paper_2303_08989_b200.network import Network
    from paper_2303_08989_b200.slicing import (SlicePlan, contraction_cost, device_evaluator,
                                               sliced_amplitude)
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cycles = args.cycles
    circ = sycamore_like(cycles, 1)
    x = [(q * 7 + 3) % 2 for q in range(circ.n_qubits)]
    spec = circuit_to_network(circ, x)
    t0 = time.perf_counter()
    path, sliced, path_kind = load_or_build_plan(spec, cycles, args.path)
    plan = SlicePlan.build(spec, path, sliced)
    plan_s = time.perf_counter() - t0
    big, macs = contraction_cost(spec, path, sliced)
    total_flops = 8.0 * macs * plan.n_slices
    _, macs_unsliced = contraction_cost(spec, path)
    width = math.log2(max(1, contraction_cost(spec, path)[0]))
    h = Handle(local)
    stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
    net = Network(h, plan.base)
    cfg = make_config()
    ev = device_evaluator(net, plan, cfg)
    group = None
    for _ in range(args.warmup):
        amp, full = sliced_amplitude(ev, plan, rank, world, group)
    barrier(world)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h.profile(True)  # device time of the slice batches (slice data resident in HBM)
    with ClockSampler(local) as clk:
        tw = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            amp, full = sliced_amplitude(ev, plan, rank, world, group)
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - tw) / args.steps * 1e3
    dev_ms, _ = h.profile_read_batches()
    h.profile(False)
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1) / args.steps, wall), world)
    ms = max_over_ranks(dev_ms / args.steps, world)
    if rank == 0:
        # fidelity: slice 0 against a complex128 contraction of the same path (GPU)
        from paper_2303_08989_b200.slicing import assignment, slice_spec
        sub = slice_spec(spec, plan.sliced, assignment(0, plan.dims))
        t1 = time.perf_counter()
        z128 = contract_c128(sub, path, dev)
        torch.cuda.empty_cache()
        fid = {"slice0_rel_err_vs_c128": float(abs(complex(full[0]) - z128) / abs(z128)),
               "reference": "complex128 contraction of slice 0 along the same path (torch)",
               "reference_s": round(time.perf_counter() - t1, 2)}
        line = {
            "metric": f"{SYC_METRIC[:-9]}, m={cycles}, {plan.n_slices} slices, AUTO-0)", "value": round(1e3 / ms, 4), "unit": "amplitudes/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c64 (AUTO-0: TF32TCEC / FP16TCEC* / FP32 tiers)",
            "data": f"synthetic circuit sycamore_like({cycles}, 1)",
            "config": {"workload": f"configs[3] class: 53-qubit Sycamore layout, {cycles} fSim cycles, "
                                   f"{plan.n_slices} slices ({len(sliced)} bonds) over {world} GPU(s)",
                       "path": f"{path_kind}, {len(path)} steps, width 2^{width:.0f} unsliced, "
                               f"2^{math.log2(big):.0f} per slice", "plan_s": round(plan_s, 2),
                       "flops_unsliced": 8.0 * macs_unsliced,
                       "flops_per_amplitude": total_flops,
                       "collective": "one all_gather of 8 B per slice (NCCL), slice-ordered f64 sum"},
            "e2e": {"value": round(1e3 / e2e_ms, 4), "unit": "amplitudes/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": int(sum(np.asarray(d).size * 8 for d in plan.run_data(0))
                                              * -(-plan.n_slices // world)),
                    "d2h_bytes_per_step": 8 * -(-plan.n_slices // world),
                    "note": "the whole step through Network.node_batch from host slice data, incl. the "
                            "cross-rank all_gather and the host f64 sum; value = device time of the batches"},
            "achieved_tflops": round(total_flops / (ms * 1e-3) / 1e12, 2),
            "amplitude": [float(amp.real), float(amp.imag)],
            "fidelity": fid, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    net.close()
    h.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


SKEWED_SHAPES = [(2048, 16384, 64), (512, 16384, 512), (512, 8192, 1024), (1024, 4096, 8192),
                 (2048, 4096, 32), (256, 16384, 64), (128, 1024, 4096)]
IRREGULAR_N = (20, 22, 24, 26)


def type3_device(rows, cols, gen, dev):
    """randtn Type-3 recipe (network.cpp:402-434): N(0, 1e-2) * 1e-6
    components with 16 planted 1.0 values -> e_max = 0 and ~29% of the components
    below 2^-28, so the selector must fall back to TF32TCEC."""
    import torch
    v = torch.randn((rows, cols, 2), generator=gen, device=dev).mul_(1e-2 * 1e-6)
    flat = v.view(-1, 2)
    idx = torch.randint(0, rows * cols, (16,), generator=gen, device=dev)
    flat[idx, 0] = 1.0
    flat[idx, 1] = 0.0
    return v.view(torch.complex64)[..., 0].contiguous()


def run_skewed(args):
    """configs[2]: contraction-shaped skewed CGEMMs (tall-skinny, small k) with a wide
    exponent range forcing the TF32TCEC fallback (policy size_auto = size_tf32 =
    min(m, n, k) so the statistics engage), plus the paper's irregular
    (2, 2^N, 2) / (2^N, 2, 2) family under the default policy (FP32 tier)."""
    import torch
    from paper_2303_08989_b200 import Handle, SelectionPolicy, make_config
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    h = Handle(local)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11 + rank)
    bpk, bps, hbm, src = peaks()
    rows_out, tot_flops, tot_ms = [], 0.0, 0.0
    cases = [(s, "type3") for s in SKEWED_SHAPES]
    cases += [((2, 1 << e, 2), "uniform") for e in IRREGULAR_N]
    cases += [((1 << e, 2, 2), "uniform") for e in IRREGULAR_N]
    with ClockSampler(local) as clk:
        for (m, n, k), rec in cases:
            if rec == "type3":
                a, b = type3_device(m, k, gen, dev), type3_device(k, n, gen, dev)
                mn = min(m, n, k)
                cfg = make_config(SelectionPolicy(size_auto=mn, size_tf32=mn))
            else:
                a = (torch.rand((m, k, 2), generator=gen, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
                b = (torch.rand((k, n, 2), generator=gen, device=dev) * 2 - 1).view(torch.complex64)[..., 0].contiguous()
                cfg = make_config()
            c = torch.empty((m, n), dtype=torch.complex64, device=dev)
            for _ in range(args.warmup):
                _, res = h.dispatch_cgemm(a, b, cfg, out=c)
            h.profile(True)
            barrier(world)
            torch.cuda.synchronize(dev)
            for _ in range(args.steps):
                h.dispatch_cgemm(a, b, cfg, out=c)
            stage, cnt = h.profile_read()
            h.profile(False)
            ms = sum(stage.values()) / max(cnt, 1)
            ms = max_over_ranks(ms, world)
            flops = 8.0 * m * n * k
            floor_bytes = 8.0 * (m * k + k * n + m * n)
            # fidelity on <= 8 sampled rows vs complex128 (and the bit-exact FP32 tier)
            ridx = torch.arange(0, m, max(1, m // 8), device=dev)[:8]
            ref = a[ridx].to(torch.complex128) @ b.to(torch.complex128)
            den = float(torch.linalg.norm(ref))
            err = float(torch.linalg.norm(c[ridx].to(torch.complex128) - ref)) / den if den else 0.0
            c32, _ = h.cgemm(a[ridx].contiguous(), b, "FP32_REF")
            err32 = float(torch.linalg.norm(c32.to(torch.complex128) - ref)) / den if den else 0.0
            del ref, c32
            tot_flops += flops
            tot_ms += ms
            rows_out.append({"m": m, "n": n, "k": k, "inputs": rec, "mode": res.line.split(",")[3],
                             "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 2),
                             "floor_gbs": round(floor_bytes / (ms * 1e-3) / 1e9, 1),
                             "floor_frac_hbm": round(floor_bytes / (ms * 1e-3) / 1e9 / hbm, 3),
                             "stages_ms": {k2: round(v / max(cnt, 1), 4) for k2, v in stage.items()},
                             "rel_err": err, "fp32_ref_rel_err": err32})
            del a, b, c
            torch.cuda.empty_cache()
    if rank == 0:
        value = world * tot_flops / (tot_ms * 1e-3) / 1e12
        line = {"metric": "skewed TCEC CGEMM TFLOP/s (useful 8mnk over the configs[2] shape set)",
                "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(tot_ms, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c64 (TF32TCEC / FP32 tiers)",
                "data": "synthetic: Type-3 wide-exponent-range (TF32 fallback) and uniform(-1,1)",
                "config": {"workload": "configs[2] skewed contraction-shaped CGEMMs + (2,2^N,2) family",
                           "timing": "device time of stats+prep+gemm stages (CUDA events)",
                           "parallelism": f"replicas x{world}"},
                "shapes": rows_out, "hbm_peak_gbs": hbm, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    h.close()


def contract_c128(spec, path, dev):
    """complex128 contraction of a NetworkSpec along an SSA path (torch on the
    GPU): the fidelity reference of the deep-circuit study.  Same label order
    as ttgt_contract (free_a | free_b, network.cpp:58-85)."""
    import torch
    live = {i: (list(ls), torch.from_numpy(np.asarray(d, np.complex64).reshape(ds if ds else [1])
                                           ).to(dev, torch.complex128).reshape(ds if ds else []))
            for i, (ls, ds, d) in enumerate(zip(spec.labels, spec.dims, spec.data))}
    nxt = len(spec.labels)
    for ia, ib in path:
        la, ta = live.pop(ia)
        lb, tb = live.pop(ib)
        shared = [l for l in la if l in lb]
        ia_ax = [la.index(l) for l in shared]
        ib_ax = [lb.index(l) for l in shared]
        t = torch.tensordot(ta, tb, dims=(ia_ax, ib_ax))
        live[nxt] = ([l for l in la if l not in shared] + [l for l in lb if l not in shared], t)
        nxt += 1
    (_, t), = live.values()
    return complex(t.reshape(-1)[0].item())


def run_rqc7x7(args):
    """configs[4]: deep-circuit fidelity study -- 7x7 rectangular RQC with increasing
    CZ depth, the reference's greedy path, AUTO-selected precision (default policy
    and a lowered policy that engages the tensor cores on more steps) against the
    FP32 baseline tier and a complex128 contraction of the same path."""
    import torch
    from paper_2303_08989_b200 import Handle, SelectionPolicy, make_config
    from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.network import Network
    from paper_2303_08989_b200.slicing import contraction_cost
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    h = Handle(local)
    depths = [int(d) for d in args.depths.split(",")]
    nbits = 10
    modes = [("AUTO-0", make_config()),
             ("AUTO-0-lowered", make_config(SelectionPolicy(size_auto=256, size_tf32=64))),
             ("FP32_BASELINE", make_config(force="FP32_REF"))]
    rows_out = []
    with ClockSampler(local) as clk:
        for depth in depths:
            circ = rqc_rectangular(7, 7, depth, 1)
            xs = bitstrings_for(49, nbits, 1)[rank::world] or bitstrings_for(49, nbits, 1)[:1]
            spec = circuit_to_network(circ, xs[0])
            net = Network(h, spec)
            path = net.greedy_path()
            big, macs = contraction_cost(spec, path)
            ref = np.array([contract_c128(circuit_to_network(circ, x), path, dev) for x in xs])
            torch.cuda.empty_cache()
            row = {"depth": depth, "steps": len(path), "max_intermediate": int(big),
                   "gflop_per_amplitude": round(8.0 * macs / 1e9, 2), "modes": {}}
            for label, cfg in modes:
                _, lines = net.contract(path, cfg, want_log=True)
                hist = {}
                for ln in lines:
                    kk = ln.split(",")[3]
                    hist[kk] = hist.get(kk, 0) + 1
                net.selector_batch(path, xs, cfg)  # capture / warm (one full pass)
                reps = max(2, args.steps // 5)
                torch.cuda.synchronize(dev)
                h.profile(True)
                t0 = time.perf_counter()
                for _ in range(reps):
                    amps = net.selector_batch(path, xs, cfg)
                e2e = (time.perf_counter() - t0) / (reps * len(xs)) * 1e3
                dev_ms, _ = h.profile_read_batches()
                h.profile(False)
                ms = dev_ms / (reps * len(xs))  # device time after the bitstring upload
                err = np.abs(amps.astype(np.complex128) - ref) / np.abs(ref)
                row["modes"][label] = {"ms_per_amplitude": round(ms, 3), "e2e_ms_per_amplitude": round(e2e, 3),
                                       "median_rel_err_vs_c128": float(np.median(err)),
                                       "max_rel_err_vs_c128": float(np.max(err)),
                                       "decisions": hist}
            a, f = row["modes"]["AUTO-0"], row["modes"]["FP32_BASELINE"]
            row["auto_speedup_vs_fp32_baseline"] = round(f["ms_per_amplitude"] / a["ms_per_amplitude"], 3)
            row["auto_err_ratio_vs_fp32_baseline"] = (round(a["median_rel_err_vs_c128"] /
                                                            f["median_rel_err_vs_c128"], 3)
                                                      if f["median_rel_err_vs_c128"] else None)
            if rank == 0 and not args.no_cpu and depth <= 12:
                thr = os.cpu_count() or 1
                bits = np.array(xs[:min(len(xs), thr)], np.uint8)
                r = rqc_reference_rate(bits, 49, 7, 7, depth, 1, thr)
                if r is not None:
                    row["cpu_reference_ms_per_amplitude"] = round(1e3 / r[0], 3)
                    row["cpu_reference_threads"] = thr
            net.close()
            rows_out.append(row)
        # beyond the reference's reach: its greedy path needs a 2^33-element
        # (69 GB) intermediate at depth 18 and 2^39 at depth 20; the sliced
        # plan search (paths.hyper_path) keeps every intermediate <= 2^28
        for depth in [int(d) for d in args.hyper_depths.split(",") if d]:
            from paper_2303_08989_b200.paths import hyper_path
            from paper_2303_08989_b200.slicing import assignment, slice_spec
            circ = rqc_rectangular(7, 7, depth, 1)
            xs = bitstrings_for(49, 4, 1)
            spec0 = circuit_to_network(circ, xs[0])
            t0 = time.perf_counter()
            path, sliced, flops, width = hyper_path(spec0, max_log2=28.0, trials=1, k=12, time_model=True)
            plan_s = time.perf_counter() - t0
            dims_of = {l: d for ls, ds in zip(spec0.labels, spec0.dims) for l, d in zip(ls, ds)}
            sdims = [dims_of[l] for l in sliced]
            nsl = int(np.prod(sdims)) if sliced else 1
            specs = [circuit_to_network(circ, x) for x in xs]
            ref = []
            for sp in specs:
                z = 0j
                for si in range(nsl):
                    z += contract_c128(slice_spec(sp, sliced, assignment(si, sdims)) if sliced else sp,
                                       path, dev)
                ref.append(z)
            ref = np.array(ref)
            torch.cuda.empty_cache()
            base = slice_spec(spec0, sliced, [0] * len(sliced)) if sliced else spec0
            var = sorted(set(i for i, ls in enumerate(spec0.labels) if set(sliced) & set(ls)) |
                         set(spec0.selector_nodes))
            runs = []
            for sp in specs:
                for si in range(nsl):
                    sub = slice_spec(sp, sliced, assignment(si, sdims)) if sliced else sp
                    runs.append([sub.data[i] for i in var])
            net = Network(h, base)
            row = {"depth": depth, "path": "hyper (sliced plan search)", "steps": len(path),
                   "slices": nsl, "width_log2": width, "gflop_per_amplitude": round(flops / 1e9, 2),
                   "plan_s": round(plan_s, 1), "modes": {}}
            for label, cfg in (modes[0], modes[2]):
                net.node_batch(path, var, runs[:nsl], cfg)  # capture / warm
                torch.cuda.synchronize(dev)
                h.profile(True)
                t0 = time.perf_counter()
                vals = net.node_batch(path, var, runs, cfg)
                e2e = (time.perf_counter() - t0) / len(xs) * 1e3
                dev_ms, _ = h.profile_read_batches()
                h.profile(False)
                ms = dev_ms / len(xs)
                amps = vals.astype(np.complex128).reshape(len(xs), nsl).sum(axis=1)
                err = np.abs(amps - ref) / np.abs(ref)
                row["modes"][label] = {"ms_per_amplitude": round(ms, 3), "e2e_ms_per_amplitude": round(e2e, 3),
                                       "median_rel_err_vs_c128": float(np.median(err)),
                                       "max_rel_err_vs_c128": float(np.max(err))}
            a, f = row["modes"]["AUTO-0"], row["modes"]["FP32_BASELINE"]
            row["auto_speedup_vs_fp32_baseline"] = round(f["ms_per_amplitude"] / a["ms_per_amplitude"], 3)
            row["auto_err_ratio_vs_fp32_baseline"] = (round(a["median_rel_err_vs_c128"] /
                                                            f["median_rel_err_vs_c128"], 3)
                                                      if f["median_rel_err_vs_c128"] else None)
            net.close()
            torch.cuda.empty_cache()
            rows_out.append(row)
    if rank == 0:
        deep_row = [r for r in rows_out if r["depth"] == depths[-1]][0]["modes"]["AUTO-0"]
        deep, deep_e2e = deep_row["ms_per_amplitude"], deep_row["e2e_ms_per_amplitude"]
        hyper_same = [r for r in rows_out if r["depth"] == depths[-1] and r.get("path", "").startswith("hyper")]
        line = {"metric": f"RCS 7x7 deep-circuit amplitude time (AUTO-0, depth {depths[-1]})",
                "value": deep, "unit": "ms/amplitude", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": deep, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "c64 (AUTO-0 tiers)",
                "data": "synthetic circuits rqc_rectangular(7, 7, d, 1), 10 bitstrings (experiments.cpp:185-196)",
                "config": {"workload": "configs[4] deep-circuit fidelity study, reference greedy path",
                           "fidelity_reference": "complex128 contraction of the same path (torch, GPU)",
                           "parallelism": f"bitstrings / {world}"},
                "e2e": {"value": deep_e2e, "unit": "ms/amplitude", "h2d_bytes_per_step": 49,
                        "d2h_bytes_per_step": 8,
                        "note": "the whole tcec_contract_selector_batch call per bitstring (host bits in, "
                                "host amplitude out); value = its device time after the upload"},
                "depths": rows_out, "clocks": clk.summary()}
        if hyper_same:
            # the same circuit through this repo's path finder
            line["with_path_search"] = {
                "ms_per_amplitude": hyper_same[0]["modes"]["AUTO-0"]["ms_per_amplitude"],
                "gflop_per_amplitude": hyper_same[0]["gflop_per_amplitude"],
                "greedy_gflop_per_amplitude": [r for r in rows_out if r["depth"] == depths[-1]][0]["gflop_per_amplitude"]}
        print(json.dumps(line), flush=True)
    h.close()


def gemm_kernel_name(m, n, kind, sm_count=148, auto=True):
    """The tcgen05 kernel an AUTO dispatch runs (resolve_gemm_variant in tcec_gemm.cu):
    the wide cta_group::2 kernel branching on the device decision when its tiles
    fill the SMs, else both single-CTA formats (the unselected one exits)."""
    wide = 2 * -(-m // 256) * -(-2 * n // 256) >= sm_count or (2 * n) // 64 >= 256
    fmt = "tf32" if kind == "TF32TCEC" else "f16"
    if wide:
        return f"tcec_gemm_wide_auto_kernel ({fmt} path)" if auto else f"tcec_gemm_wide_kernel<{fmt}>"
    return f"tcec_gemm_kernel<{fmt}>"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", choices=["cgemm", "rqc", "sycamore", "skewed", "rqc7x7"], default="cgemm")
    p.add_argument("--cycles", type=int, default=12)
    p.add_argument("--path", choices=["plan", "hyper", "greedy"], default="plan")
    p.add_argument("--depths", default="4,8,12,14,16")
    p.add_argument("--hyper-depths", default="16,18,20,24")
    p.add_argument("--slices-log2", type=int, default=6)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=N_DEFAULT)
    p.add_argument("--no-sweep", dest="sweep", action="store_false")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=12.0)
    p.add_argument("--ref-step-s", type=float, default=8.0)
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload == "rqc":
        run_rqc(args)
    elif args.workload == "sycamore":
        run_sycamore(args)
    elif args.workload == "skewed":
        run_skewed(args)
    elif args.workload == "rqc7x7":
        run_rqc7x7(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
