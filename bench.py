#!/usr/bin/env python
"""bench.py -- TCEC CGEMM TFLOP/s (+ fidelity) and sliced RCS time on B200
(BASELINE.json: "TCEC CGEMM TFLOP/s + fidelity; RCS contraction time at 1/2/4/8 GPUs").

Default line (one "step" = one AUTO-0 dispatch_cgemm of configs[1]'s top point,
m = n = k = 16384, on the reference's own inputs -- Rng(1 + n), A then B,
uniform_pm1f, experiments.cpp:76-83 -- with precsel.cpp:225-322 semantics:
device exponent statistics -> selection -> scale+split -> tcgen05 TCEC CGEMM
-> descale):

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value      = useful 8mnk flops / device time (CUDA events on the handle stream), inputs
             resident in HBM; N > 1 runs N replicas (the standalone CGEMM does not shard,
             SURVEY.md 8(e)) -> whole-job flops / max-over-ranks time.  `--gpus N` outside
             torchrun re-executes itself under torch.distributed.run (one rank per GPU).
e2e        = the same through tcec_dispatch_cgemm_host (H2D of A and B + dispatch + D2H of C
             inside the timed region), from pinned buffers and from pageable ones.
roofline   = the dominant kernel (the tcgen05 TCEC GEMM), 3 x 8mnk tensor-pipe flops per
             launch over its CUDA-event duration, against the measured dense bf16/fp16 peak.
cpu_baseline / decision_parity = the unmodified reference (oracle/_ref) on the same operands:
             its exp_stats_staged + select_mode over all of A and B give the decision line that
             must equal the device's byte for byte (exit 3 otherwise), then its kernels on a
             bounded row block over all host threads, extrapolated.
sliced_rcs = configs[3]: Sycamore-class 53q m=12 amplitude, slices sharded round-robin over
             the N ranks, one NCCL all_gather, slice-ordered f64 sum (every N).
legs       = (N = 1) compact configs[0] (4x4 RQC, bit-identity to the reference), configs[2]
             (skewed shapes, HBM-floor fractions), configs[4] (7x7 d16, AUTO vs FP32 tier
             against the CPU FP64 oracle).
--impl reference = the reference's own dispatch_cgemm on the same config (rank 0 only).
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


def tf32_peak():
    """Dense TF32 peak for the TF32TCEC path: half the measured dense bf16 burst
    peak of MEASURED_PEAKS.json (sm_100 tensor cores run TF32 at half the
    bf16/fp16 rate: B200_PROFILING.md 1.1 vs 2.25 PFLOP/s dense).  The cuBLAS
    TF32 8192^3 figure of profiles/r02_tf32_peak.json (tools/peak_tf32.py) is
    quoted next to it: cuBLAS's TF32 kernel does not reach the hardware rate on
    this pool (the TCEC kernel runs above it), so it cannot be the bound.
    Fallback: B200_PROFILING.md's 1.1 PF dense."""
    bpk, _, _, src = peaks()
    cub = ""
    p = os.path.join(ROOT, "profiles", "r02_tf32_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))["tf32"]
        cub = (f"; cuBLAS TF32 8192^3 on the same pool: {d['burst_tflops']} burst / "
               f"{d['sustained_tflops']} sustained (profiles/r02_tf32_peak.json)")
    if src == "measured":
        return round(bpk / 2, 1), (f"measured dense bf16 burst {bpk} TFLOP/s (MEASURED_PEAKS.json) / 2 "
                                   f"= the dense TF32 rate (1:2 on sm_100, B200_PROFILING.md){cub}")
    return 1100.0, "B200_PROFILING.md fallback: 1.1 PFLOP/s dense TF32" + cub


def frac_at_clock(achieved_tflops, tf32, clk):
    """achieved / the dense tensor rate at the median SM clock of the run (TF32
    4096, FP16/BF16 8192 flop/clk/SM on sm_100: 1.1 / 2.25 PF at ~1.85 GHz)."""
    try:
        mhz = clk.summary().get("sm_mhz")
    except Exception:
        mhz = None
    if not mhz:
        return None
    return round(achieved_tflops * 1e12 / (148 * (4096 if tf32 else 8192) * mhz * 1e6), 4)


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
def _ref_dispatch_fn():
    """oracle/_ref's bridge onto the reference's own dispatch_cgemm selection +
    row-partitioned kernels (ref_dispatch_rows_threaded_timed), or None."""
    import oracle as O
    ref = O.reference()
    if ref is None:
        return None, None
    fn = ref.lib.ref_dispatch_rows_threaded_timed
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                   C.c_int64, C.POINTER(O.ConfigPod), C.c_int, C.c_char_p, C.c_int,
                   C.POINTER(C.c_int), C.POINTER(C.c_double)]
    fn.restype = C.c_int
    return fn, O


def reference_dispatch_sample(a_host, b_host, rows, threads):
    """The reference's dispatch_cgemm (precsel.cpp:225-322, default policy) on
    the full operands -- exp_stats_staged of all of A and B, matrix_tolerance,
    select_mode, DecisionRecord::to_line -- with the selected kind's CGEMM
    timed on output rows [0, rows) over `threads` host threads (row
    partitioning is bit-identical, kernels.hpp:16-19).  Returns
    (decision line, [stats_s, prep_s, gemm_s]) or None without oracle/_ref."""
    fn, O = _ref_dispatch_fn()
    if fn is None:
        return None
    m, k = a_host.shape
    n = b_host.shape[1]
    c = np.empty((max(rows, 1), n), np.complex64)
    line = C.create_string_buffer(256)
    kind = C.c_int(0)
    t = (C.c_double * 3)()
    cfg = O.make_config()
    rc = fn(a_host.ctypes.data, b_host.ctypes.data, c.ctypes.data, m, n, k, 0, rows, C.byref(cfg),
            threads, line, 256, C.byref(kind), t)
    if rc:
        raise RuntimeError(f"reference dispatch failed (rc={rc})")
    return line.value.decode(), [t[0], t[1], t[2]]


def calibrate_rows(a_host, b_host, budget_s, threads):
    """Rows of the bounded CPU sample: the row GEMM of `threads` rows timed
    once, scaled to about budget_s of GEMM work."""
    r = reference_dispatch_sample(a_host, b_host, threads, threads)
    if r is None:
        return None
    per_row = r[1][2] / threads
    m = a_host.shape[0]
    rows = int(max(threads, min(m, budget_s / max(per_row, 1e-9))))
    return max(threads, (rows // threads) * threads)


# ---------------------------------------------------------------- helpers
def dist_setup(gpus=None):
    """One process per GPU (RANK / LOCAL_RANK / WORLD_SIZE from torchrun);
    idempotent so the legs of one run share the process group."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TCEC_BENCH_SHARED_GPU=1: every rank on cuda:0 with gloo -- exercises the
    # N > 1 code path on a one-GPU box (NCCL refuses two ranks on one GPU);
    # never used for a reported number
    shared = os.environ.get("TCEC_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if shared and not dist.is_initialized():
            dist.init_process_group("gloo")
            return world, rank, local
        # NCCL's own log stays on (transport / NVLS lines), in files next to the run
        logdir = os.path.join(ROOT, "gpurun_out")
        os.makedirs(logdir, exist_ok=True)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, "nccl.%h.%p.log"))
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def dist_teardown(world):
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


INPUTS_NOTE = ("reference inputs: one Rng(1 + n) (std::mt19937_64), A then B, two uniform_pm1f "
               "draws per complex element (experiments.cpp:76-83, rng.hpp:35)")


def workload_name(n):
    return (f"configs[1] CGEMM sweep top: m=n=k={n}, AUTO-0 dispatch_cgemm (default "
            f"SelectionPolicy: device statistics -> selection -> scale+split -> TCEC GEMM)")


def host_inputs(n):
    """configs[1] operands exactly as run_gemm_bench makes them (pinned host)."""
    from paper_2303_08989_b200.workload import sweep_operands
    return sweep_operands(n, seed=1)


# ------------------------------------------------------------------- arms
def cgemm_headline(args, world, rank, local):
    """configs[1] top point on every rank (replicas); returns rank 0's line."""
    import torch
    from paper_2303_08989_b200 import Handle, make_config
    dev = torch.device("cuda", local)
    n = args.n
    h = Handle(local)
    stream = torch.cuda.ExternalStream(h.stream_ptr, device=dev)
    t_gen = time.perf_counter()
    a_h, b_h = host_inputs(n)
    t_gen = time.perf_counter() - t_gen
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

    # ---- end to end through the host-buffer C-ABI (pinned, then pageable)
    a_np, b_np = a_h.numpy(), b_h.numpy()
    c_h = torch.empty((n, n), dtype=torch.complex64, pin_memory=True)
    c_np = c_h.numpy()

    def e2e_run(an, bn, cn, steps):
        h.dispatch_cgemm_host(an, bn, cfg, out=cn)  # allocate staging once
        barrier(world)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(steps):
            h.dispatch_cgemm_host(an, bn, cfg, out=cn)
        e1.record(stream)
        e1.synchronize()
        return max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / steps,
                              world)

    e2e_ms = e2e_run(a_np, b_np, c_np, args.steps)
    pipe_runs, pipe_reruns = h.host_pipeline_stats()
    e2e_pageable_ms = None
    if args.pageable and world == 1:
        # the drop-in's std::vector storage is pageable: same call on plain numpy copies
        a_pg, b_pg = np.array(a_np, copy=True), np.array(b_np, copy=True)
        c_pg = np.empty_like(c_np)
        e2e_pageable_ms = e2e_run(a_pg, b_pg, c_pg, max(2, args.steps // 2))
        del a_pg, b_pg, c_pg

    # ---- fidelity: sampled rows vs complex128, and the bit-exact FP32 tier on the same rows
    rows = torch.from_numpy(np.random.default_rng(3).choice(n, 16, replace=False)).to(dev)
    ref = a[rows].to(torch.complex128) @ b.to(torch.complex128)
    err = float(torch.linalg.norm(c[rows].to(torch.complex128) - ref) / torch.linalg.norm(ref))
    c32, _ = h.cgemm(a[rows].contiguous(), b, "FP32_REF")
    err32 = float(torch.linalg.norm(c32.to(torch.complex128) - ref) / torch.linalg.norm(ref))
    del ref

    # ---- small sweep (configs[1] 1024..8192 on the reference inputs), AUTO and forced formats
    sweep, sweep_ops = {}, {}
    if args.sweep and rank == 0:
        for sn in (1024, 2048, 4096, 8192):
            sa_h, sb_h = host_inputs(sn)
            sweep_ops[sn] = (sa_h.numpy(), sb_h.numpy())
            sa, sb = sa_h.to(dev), sb_h.to(dev)
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
                    row["AUTO-0 decision"] = r.line
            sweep[str(sn)] = row
            del sa, sb, sc

    # ---- CPU baseline (rank 0, N=1 only): the reference's own dispatch on the
    # same operands -- its decision line must equal the device's byte for byte
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        thr = os.cpu_count() or 1
        rows_s = calibrate_rows(a_np, b_np, args.cpu_budget, thr)
        if rows_s is not None:
            ref_line, (st_s, prep_s, gemm_s) = reference_dispatch_sample(a_np, b_np, rows_s, thr)
            full_s = st_s + prep_s + gemm_s * n / rows_s
            parity = {str(n): {"reference": ref_line, "device": decision,
                               "identical": ref_line == decision}}
            for sn, (sa_np, sb_np) in sweep_ops.items():
                rl, _ = reference_dispatch_sample(sa_np, sb_np, 0, thr)
                parity[str(sn)] = {"reference": rl, "device": sweep[str(sn)]["AUTO-0 decision"],
                                   "identical": rl == sweep[str(sn)]["AUTO-0 decision"]}
            cpu = {"value": round(flops / full_s / 1e12, 6), "unit": "TFLOP/s", "cores": thr,
                   "kind": "reference",
                   "sample": f"the reference's dispatch_cgemm on the same operands: exp_stats_staged "
                             f"+ select_mode over all of A and B ({st_s:.1f} s), scale+split "
                             f"({prep_s:.1f} s), {kind} rows 0..{rows_s} with its kernels on {thr} "
                             f"threads ({gemm_s:.1f} s), row GEMM extrapolated to all {n} rows"}
    del sweep_ops

    line = None
    if rank == 0:
        bpk, bps, hbm, src = peaks()
        tensor_flops = 3.0 * flops  # hi*hi, lo*hi, hi*lo tensor-core products per launch
        achieved = tensor_flops / (gemm_ms * 1e-3) / 1e12
        tf32 = kind == "TF32TCEC"
        if tf32:
            peak, psrc = tf32_peak()
        else:
            peak, psrc = bps, f"{src} dense bf16 sustained (MEASURED_PEAKS.json; fp16 = bf16 rate)"
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"tcec_gemm_{'tf32' if tf32 else 'f16'}_n{n}")
        value = world * flops / (ms_max * 1e-3) / 1e12
        e2e = {"value": round(world * flops / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
               "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * n * 8,
               "host_buffers": "pinned",
               "pipeline": {"runs": pipe_runs, "reruns": pipe_reruns,
                            "note": "H2D of B column parts / A row chunks overlapped with the GEMM "
                                    "blocks under a decision from the first parts, checked against "
                                    "the exact one (reruns = recomputed on disagreement)"}}
        if e2e_pageable_ms:
            e2e["pageable"] = {"value": round(world * flops / (e2e_pageable_ms * 1e-3) / 1e12, 2),
                               "unit": "TFLOP/s",
                               "note": "same call from pageable numpy buffers (the C++ drop-in's "
                                       "std::vector storage): staged through a pinned ring"}
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(value / PAPER_A100_FP16TCEC, 2),
            "baseline_ref": "54.2 TFLOP/s FP16TCEC CGEMM max on A100 (PAPER.md:246)",
            "dtype": f"c64 (FP32-level via error-corrected {'TF32' if tf32 else 'FP16'} products)",
            "data": "synthetic, the reference's own generator, resident in HBM",
            "config": {"workload": workload_name(n), "decision": decision, "inputs": INPUTS_NOTE},
            "parallelism": f"replicas x{world} (the standalone CGEMM does not shard, SURVEY 8(e))",
            "l2": "inputs (2 GiB per operand) exceed the 126 MB L2",
            "flush_kblocks": h.flush_kblocks, "input_generation_s": round(t_gen, 2),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": gemm_kernel_name(n, n, kind),
                         "frac_at_clock": frac_at_clock(achieved, tf32, clk),
                         "note": f"3 x 8mnk tensor-pipe flops per launch / CUDA-event time; "
                                 f"peak = {psrc}; frac_at_clock = achieved / (148 SMs x "
                                 f"{4096 if tf32 else 8192} dense flop/clk/SM x the median SM clock "
                                 f"sampled under load): the tensor pipe's share at the clock the "
                                 f"power cap left"},
            "stages_ms": {k2: round(v / max(cnt, 1), 3) for k2, v in stage.items()},
            "fidelity": {"rel_err": err, "fp32_ref_rel_err": err32,
                         "ratio_vs_fp32": round(err / err32, 3) if err32 else None,
                         "sample": "16 random rows vs complex128"},
            "e2e": e2e,
            # per AUTO dispatch: stats1, stats2 (whose last block runs the
            # selection), prep_a, prep_b and ONE tcgen05 GEMM (the wide kernel
            # branches on the device decision), plus a cudaMemsetAsync of the
            # decision slot
            "gpu_launches": 5 * args.steps,
            "clocks": clk.summary(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if parity:
            line["decision_parity"] = parity
        if sweep:
            line["sweep_tflops"] = sweep
    h.close()
    del a, b, c
    torch.cuda.empty_cache()
    return line


def run_ours(args):
    """The default line: the configs[1] headline (replicas over the ranks),
    the sliced Sycamore-class RCS (configs[3], slices sharded over the ranks,
    one NCCL all_gather) and, at N = 1, compact legs of configs[0], [2], [4]."""
    world, rank, local = dist_setup(args.gpus)
    line = cgemm_headline(args, world, rank, local)
    syc = None
    if args.sliced:
        sub = argparse.Namespace(**vars(args))
        sub.steps, sub.warmup = args.sliced_steps, 3
        syc = run_sycamore(sub, emit=False)
    legs = {}
    if world == 1 and args.legs:
        sub = argparse.Namespace(**vars(args))
        sub.steps, sub.warmup = 5, 3
        for name, fn in (("configs[0]_rqc4x4", run_rqc), ("configs[2]_skewed", run_skewed),
                         ("configs[4]_rqc7x7_d16", run_rqc7x7_leg)):
            t0 = time.perf_counter()
            try:
                legs[name] = fn(sub, emit=False)
            except Exception as e:  # a leg must not take the headline down
                legs[name] = {"error": f"{type(e).__name__}: {e}"}
            if isinstance(legs[name], dict):
                legs[name]["leg_s"] = round(time.perf_counter() - t0, 1)
    if rank == 0:
        if syc:
            line["sliced_rcs"] = syc
        if legs:
            line["legs"] = legs
        print(json.dumps(line), flush=True)
    dist_teardown(world)
    if rank == 0 and line.get("decision_parity"):
        bad = [k for k, v in line["decision_parity"].items() if not v["identical"]]
        if bad:
            print(f"DECISION PARITY FAILED for n = {bad}", file=sys.stderr, flush=True)
            sys.exit(3)


def run_reference(args):
    """The reference's own CPU path on the same config: its dispatch_cgemm
    (statistics + selection over all of A and B, then the selected kind) on
    the same inputs, the row GEMM timed on a bounded row block over all host
    threads and extrapolated.  Rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.n
    a_h, b_h = host_inputs(n)
    a_np, b_np = a_h.numpy(), b_h.numpy()
    thr = os.cpu_count() or 1
    rows = calibrate_rows(a_np, b_np, args.ref_step_s, thr)
    if rows is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the reference build) "
                          "is missing on this machine"}), flush=True)
        return
    for _ in range(args.warmup):
        reference_dispatch_sample(a_np, b_np, rows, thr)
    vals, wall, ref_line = [], 0.0, None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref_line, (st_s, prep_s, gemm_s) = reference_dispatch_sample(a_np, b_np, rows, thr)
        wall += time.perf_counter() - t0
        vals.append(st_s + prep_s + gemm_s * n / rows)
    full_s = float(np.mean(vals))
    value = 8.0 * n * n * n / full_s / 1e12
    kind = ref_line.split(",")[3]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(full_s * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c64 (FP32-level via error-corrected FP16 products)",
        "data": "synthetic, the reference's own generator, resident in HBM",
        "config": {"workload": workload_name(n), "decision": ref_line, "inputs": INPUTS_NOTE},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": thr, "kind": "reference",
                         "sample": f"per step: the unmodified reference's dispatch_cgemm selection "
                                   f"(exp_stats_staged + matrix_tolerance + select_mode over all of "
                                   f"A and B), then {kind} on rows 0..{rows} of C with its kernels "
                                   f"over {thr} threads; the row GEMM extrapolated to all {n} rows "
                                   f"({wall / args.steps:.1f} s wall per step)"},
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


def run_rqc(args, emit=True):
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
        from paper_2303_08989_b200.network import statevector_oracle
        sv = statevector_oracle(h, circ).cpu().numpy()  # the reference's f64 oracle, on the device
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
        if emit:
            print(json.dumps(line), flush=True)
    net.close()
    h.close()
    if not emit:
        return _compact_leg(line) if rank == 0 else None


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


def run_sycamore(args, emit=True):
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
        onet = Network(h, sub)
        z64 = complex(onet.contract_oracle(path).data.reshape(-1)[0])
        onet.close()
        torch.cuda.empty_cache()
        fid = {"slice0_rel_err_vs_f64_oracle": float(abs(complex(full[0]) - z64) / abs(z64)),
               "reference": "contract_network_oracle of slice 0 along the same path (network.cpp:179-186; "
                            "f64 fold on the device, bit-identical to the reference's CPU oracle)",
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
        if emit:
            print(json.dumps(line), flush=True)
    net.close()
    h.close()
    torch.cuda.empty_cache()
    if emit:
        dist_teardown(world)
        return None
    return _compact_leg(line) if rank == 0 else None


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


def run_skewed(args, emit=True):
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
        if emit:
            print(json.dumps(line), flush=True)
    h.close()
    if not emit:
        return _compact_leg(line) if rank == 0 else None


def contract_f64(h, spec, path):
    """contract_network_oracle (network.cpp:179-186) of a closed network along
    `path`: the f64 fold on the device, bit-identical to the reference's CPU
    oracle -- the fidelity reference of the deep-circuit legs."""
    from paper_2303_08989_b200.network import Network
    onet = Network(h, spec)
    try:
        return complex(onet.contract_oracle(path).data.reshape(-1)[0])
    finally:
        onet.close()


def _compact_leg(line):
    """A sub-workload's JSON line without the per-run boilerplate."""
    if not line:
        return None
    drop = {"steps", "warmup", "higher_is_better", "vs_baseline", "n_gpus", "clocks", "dtype", "data",
            "hbm_peak_gbs"}
    out = {k: v for k, v in line.items() if k not in drop}
    if "shapes" in out:
        out["shapes"] = [{k: r[k] for k in ("m", "n", "k", "inputs", "mode", "ms", "tflops",
                                            "floor_frac_hbm", "rel_err", "fp32_ref_rel_err") if k in r}
                         for r in out["shapes"]]
    return out


def run_rqc7x7_leg(args, emit=False):
    """configs[4] deep point (7x7, depth 16) on the reference's greedy path:
    AUTO-0 vs the FP32 baseline tier per amplitude, errors against the CPU
    FP64 contraction oracle (contract_network_oracle, network.cpp:179-186) of
    the same path and bitstrings (the checker, timed on the host)."""
    import torch
    from paper_2303_08989_b200 import Handle, make_config
    from paper_2303_08989_b200.circuits import bitstrings_for, circuit_to_network, rqc_rectangular
    from paper_2303_08989_b200.network import Network
    from paper_2303_08989_b200.slicing import contraction_cost
    world, rank, local = dist_setup(args.gpus)
    if rank != 0:
        return None
    dev = torch.device("cuda", local)
    h = Handle(local)
    depth, nb = 16, 3
    circ = rqc_rectangular(7, 7, depth, 1)
    xs = bitstrings_for(49, 10, 1)[:nb]  # experiments.cpp:185-196
    spec = circuit_to_network(circ, xs[0])
    net = Network(h, spec)
    path = net.greedy_path()
    big, macs = contraction_cost(spec, path)
    out = {"metric": "7x7 RQC depth-16 amplitude time (reference greedy path)", "unit": "ms/amplitude",
           "steps_per_amplitude": len(path), "gflop_per_amplitude": round(8.0 * macs / 1e9, 1),
           "max_intermediate": int(big), "bitstrings": nb, "modes": {}}
    amps_by = {}
    for label, cfg in (("AUTO-0", make_config()), ("FP32_BASELINE", make_config(force="FP32_REF"))):
        net.selector_batch(path, xs, cfg)  # capture / warm
        torch.cuda.synchronize(dev)
        h.profile(True)
        t0 = time.perf_counter()
        reps = 2
        for _ in range(reps):
            amps = net.selector_batch(path, xs, cfg)
        e2e = (time.perf_counter() - t0) / (reps * nb) * 1e3
        dev_ms, _ = h.profile_read_batches()
        h.profile(False)
        amps_by[label] = amps.astype(np.complex128)
        out["modes"][label] = {"ms_per_amplitude": round(dev_ms / (reps * nb), 3),
                               "e2e_ms_per_amplitude": round(e2e, 3)}
    net.close()
    h.close()
    out["value"] = out["modes"]["AUTO-0"]["ms_per_amplitude"]
    out["auto_speedup_vs_fp32_baseline"] = round(out["modes"]["FP32_BASELINE"]["ms_per_amplitude"]
                                                 / out["value"], 3)
    # fidelity reference: contract_network_oracle (network.cpp:179-186) of the
    # same path, the f64 fold on the device -- bit-identical to the reference's
    # CPU oracle (tests/test_gpu_network.py::test_device_f64_oracle_is_the_reference_oracle)
    t0 = time.perf_counter()
    h = Handle(local)
    zref = []
    for x in xs:
        onet = Network(h, circuit_to_network(circ, x))
        zref.append(complex(onet.contract_oracle(path).data.reshape(-1)[0]))
        onet.close()
    h.close()
    zref = np.array(zref)
    for label, amps in amps_by.items():
        err = np.abs(amps - zref) / np.abs(zref)
        out["modes"][label]["median_rel_err_vs_f64_oracle"] = float(np.median(err))
        out["modes"][label]["max_rel_err_vs_f64_oracle"] = float(np.max(err))
    fa = out["modes"]["FP32_BASELINE"]["median_rel_err_vs_f64_oracle"]
    out["auto_err_ratio_vs_fp32_baseline"] = (round(out["modes"]["AUTO-0"]["median_rel_err_vs_f64_oracle"]
                                                    / fa, 3) if fa else None)
    out["fidelity_reference"] = {"what": "contract_network_oracle of the same greedy path, f64 on the device "
                                         "(bit-identical to the reference's CPU oracle)",
                                 "seconds": round(time.perf_counter() - t0, 2), "bitstrings": nb}
    return out


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
            ref = np.array([contract_f64(h, circuit_to_network(circ, x), path) for x in xs])
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
                                       "median_rel_err_vs_f64_oracle": float(np.median(err)),
                                       "max_rel_err_vs_f64_oracle": float(np.max(err)),
                                       "decisions": hist}
            a, f = row["modes"]["AUTO-0"], row["modes"]["FP32_BASELINE"]
            row["auto_speedup_vs_fp32_baseline"] = round(f["ms_per_amplitude"] / a["ms_per_amplitude"], 3)
            row["auto_err_ratio_vs_fp32_baseline"] = (round(a["median_rel_err_vs_f64_oracle"] /
                                                            f["median_rel_err_vs_f64_oracle"], 3)
                                                      if f["median_rel_err_vs_f64_oracle"] else None)
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
                    z += contract_f64(h, slice_spec(sp, sliced, assignment(si, sdims)) if sliced else sp,
                                      path)
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
                                       "median_rel_err_vs_f64_oracle": float(np.median(err)),
                                       "max_rel_err_vs_f64_oracle": float(np.max(err))}
            a, f = row["modes"]["AUTO-0"], row["modes"]["FP32_BASELINE"]
            row["auto_speedup_vs_fp32_baseline"] = round(f["ms_per_amplitude"] / a["ms_per_amplitude"], 3)
            row["auto_err_ratio_vs_fp32_baseline"] = (round(a["median_rel_err_vs_f64_oracle"] /
                                                            f["median_rel_err_vs_f64_oracle"], 3)
                                                      if f["median_rel_err_vs_f64_oracle"] else None)
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
                           "fidelity_reference": "contract_network_oracle of the same path (f64 fold on the device, bit-identical to the reference's CPU oracle)",
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


def spawn_ranks(gpus):
    """`python bench.py --gpus N` outside torchrun: re-exec this command under
    torch.distributed.run with N local ranks (one process per GPU, NCCL,
    rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # NCCL's own log (NVLS / NVLink transport lines)
    logdir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(logdir, exist_ok=True)
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, "nccl.%h.%p.log"))
    # "--" ends torchrun's own options, so none of ours is taken as an
    # abbreviation of one of its flags
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "--", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd, env=env)


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
    p.add_argument("--no-sliced", dest="sliced", action="store_false",
                   help="skip the sliced Sycamore-class RCS object of the default line")
    p.add_argument("--sliced-steps", type=int, default=3)
    p.add_argument("--no-legs", dest="legs", action="store_false",
                   help="skip the configs[0]/[2]/[4] legs of the default line (N = 1)")
    p.add_argument("--no-pageable", dest="pageable", action="store_false")
    p.add_argument("--cpu-budget", type=float, default=12.0)
    p.add_argument("--ref-step-s", type=float, default=4.0)
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference" and args.workload in ("sycamore", "skewed", "rqc7x7"):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the reference has no {args.workload} CPU arm beyond the default line"}))
        return
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
