"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    make -C oracle all ref && python tests/golden/make_golden.py

Every output value below comes from oracle/_ref/libmpsgemm_ref.so, i.e. the
unmodified reference sources compiled in place (oracle/ref_bridge.cpp calls the
reference's public API).  Inputs are regenerated from seeds with the
reference's Rng (pinned in rng.json), so the fixtures stay small.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from tests.golden.recipes import SPECIALS, matrix_recipe, random_bits  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def main():
    ref = O.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libmpsgemm_ref.so missing: run make -C oracle ref")
    lib = ref.lib

    # ------------------------------------------------------------ rng pin
    lib.ref_rng_stream.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.POINTER(C.c_double)]
    lib.ref_rng_uniform_c32.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_float)]
    rng = {}
    for seed in (1, 42, 1 ^ 0xC2B2AE3D27D4EB4F):
        for kind in (0, 1, 2, 3):
            out = np.zeros(64, dtype=np.float64)
            lib.ref_rng_stream(seed, kind, 64, out.ctypes.data_as(C.POINTER(C.c_double)))
            rng[f"{seed}:{kind}"] = out.tolist()
        m = np.zeros((4, 5), dtype=np.complex64)
        lib.ref_rng_uniform_c32(seed, 4, 5, m.view(np.float32).ctypes.data_as(C.POINTER(C.c_float)))
        rng[f"{seed}:uniform_c32"] = bits(m.view(np.float32)).tolist()
    json.dump(rng, open(os.path.join(OUT, "rng.json"), "w"))

    # ----------------------------------------------------- lowprec vectors
    x = np.concatenate([np.array(SPECIALS, dtype=np.float32), random_bits(7, 8192)])
    low = {"x": bits(x)}
    for fmt in (0, 1):
        for rd in (0, 1):
            q, ovf = ref.quantize_buf(x, fmt, rd)
            low[f"q{fmt}{rd}"] = bits(q)
            low[f"q{fmt}{rd}_ovf"] = np.array([ovf])
            # per-element overflow flags for the special values
            low[f"q{fmt}{rd}_ovf_each"] = np.array(
                [ref.quantize_buf(np.array([v], np.float32), fmt, rd)[1] for v in SPECIALS])
        hi, lo, ovf = ref.split_buf(x, fmt)
        low[f"hi{fmt}"], low[f"lo{fmt}"], low[f"s{fmt}_ovf"] = bits(hi), bits(lo), np.array([ovf])
    for s in (0, 1, -7, 34, -163, 163, 1100):
        low[f"scale{s}"] = bits(ref.scale_buf(x, s))
    np.savez_compressed(os.path.join(OUT, "lowprec.npz"), **low)

    # --------------------------------------------------- stats / selection
    stats = []
    for name in ("uniform", "tiny20", "huge20", "banded", "type3", "zeros", "subnormal",
                 "mixed40", "ones", "sparse"):
        for (rows, cols, seed) in ((4, 4, 1), (37, 29, 2), (128, 96, 3)):
            m = matrix_recipe(name, rows, cols, seed)
            rec = {"recipe": name, "rows": rows, "cols": cols, "seed": seed,
                   "full": ref.exp_stats(m).as_dict(), "staged": {}, "level": {}}
            for t in (0.0, 0.1, 0.5, 0.95, 1.0):
                st = ref.exp_stats_staged(m, 14, t)
                rec["staged"][str(t)] = st.as_dict()
                rec["level"][str(t)] = ref.matrix_tolerance(st, t, 14)
            stats.append(rec)
    sel = []
    for la in (0, 1, 2):
        for lb in (0, 1, 2):
            for ea in (None, -20, 0, 3):
                for eb in (None, -40, 0, 14):
                    kind, sa, sb = ref.select_mode(la, ea, lb, eb, 14)
                    sel.append({"la": la, "ea": ea, "lb": lb, "eb": eb, "kind": kind, "sa": sa,
                                "sb": sb})
    json.dump({"stats": stats, "select": sel}, open(os.path.join(OUT, "precsel.json"), "w"))

    # -------------------------------------------------------------- cgemm
    cg = {}
    shapes = [(1, 1, 1), (3, 5, 7), (8, 32, 16), (13, 37, 65), (16, 48, 33), (64, 64, 64),
              (100, 1, 50), (1, 200, 3)]
    for (m, n, k) in shapes:
        a = matrix_recipe("uniform", m, k, 1000 + m)
        b = matrix_recipe("uniform", k, n, 2000 + n)
        for mode in O.MODES:
            c, ovf = ref.cgemm(a, b, mode)
            cg[f"{m}x{n}x{k}:{mode}"] = bits(c.view(np.float32))
        cg[f"{m}x{n}x{k}:oracle"] = ref.cgemm_oracle(a, b).view(np.float64)
    np.savez_compressed(os.path.join(OUT, "cgemm.npz"), **cg)

    # ----------------------------------------------------------- dispatch
    disp = []
    cases = [
        ("uniform", "uniform", dict()),
        ("uniform", "uniform", dict(size_auto=16, size_tf32=8)),
        ("uniform", "uniform", dict(size_auto=16, size_tf32=8, threshold_t=0.1)),
        ("tiny20", "tiny20", dict(size_auto=16, size_tf32=8)),
        ("banded", "banded", dict(size_auto=16, size_tf32=8)),
        ("type3", "uniform", dict(size_auto=16, size_tf32=8)),
        ("type3", "uniform", dict(size_auto=16, size_tf32=8, threshold_t=0.5)),
        ("huge20", "banded", dict(size_auto=16, size_tf32=8)),
        ("zeros", "uniform", dict(size_auto=16, size_tf32=8)),
        ("uniform", "uniform", dict(size_auto=1 << 40, size_tf32=16)),
    ] + [("uniform", "tiny20", dict(force=f)) for f in O.FORCED]
    for ia, (ra, rb, kw) in enumerate(cases):
        for (m, n, k) in ((48, 40, 32), (17, 33, 20)):
            a = matrix_recipe(ra, m, k, 300 + ia)
            b = matrix_recipe(rb, k, n, 400 + ia)
            cfg = O.make_config(**kw)
            rc, c, res = ref.dispatch_cgemm(a, b, cfg)
            disp.append({"a": ra, "b": rb, "seed_a": 300 + ia, "seed_b": 400 + ia, "m": m, "n": n,
                         "k": k, "cfg": kw, "rc": rc, "kind": O.KINDS[res.kind],
                         "scale_a": res.scale_a, "scale_b": res.scale_b,
                         "overflow": res.overflow, "line": res.line.decode(),
                         "c_bits_sha": hashlib.sha256(bits(c.view(np.float32)).tobytes()).hexdigest(),
                         "c_oracle": ref.cgemm_oracle(a, b).view(np.float64).tolist()
                         if m * n <= 400 else None})
    json.dump(disp, open(os.path.join(OUT, "dispatch.json"), "w"))

    # ------------------------------------------------------------ permute
    perm = {}
    prng = np.random.default_rng(5)
    for case in range(12):
        r = int(prng.integers(1, 7))
        dims = [int(d) for d in prng.integers(1, 5, r)]
        axis = [int(v) for v in prng.permutation(r)]
        t = matrix_recipe("uniform", 1, int(np.prod(dims)), 700 + case).reshape(dims)
        out = ref.permute(t, axis)
        perm[f"{case}"] = {"dims": dims, "axis": axis,
                           "out": bits(out.reshape(-1).view(np.float32)).tolist()}
    json.dump(perm, open(os.path.join(OUT, "permute.json"), "w"))

    # ---------------------------------------------------------- circuits
    lib.ref_rqc_circuit_text.restype = C.c_int64
    lib.ref_rqc_circuit_text.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_char_p, C.c_int64]
    lib.ref_rqc_network_text.restype = C.c_int64
    lib.ref_rqc_network_text.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64,
                                         C.POINTER(C.c_uint8), C.c_char_p, C.c_int64]
    lib.ref_rqc_path.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int), C.c_int]
    lib.ref_rqc_amplitude.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_uint8),
                                      C.POINTER(O.ConfigPod), C.POINTER(C.c_float),
                                      C.POINTER(C.c_double), C.c_char_p, C.c_int64]
    lib.ref_rqc_amplitude_tn_oracle.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
    lib.ref_rqc_amplitude_sv_oracle.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
    from paper_2303_08989_b200.circuits import bitstrings_for
    rq = []
    for (rows, cols, depth, seed) in ((2, 2, 4, 5), (2, 3, 6, 21), (4, 4, 8, 1), (4, 4, 12, 1)):
        nq = rows * cols
        need = lib.ref_rqc_circuit_text(rows, cols, depth, seed, None, 0)
        buf = C.create_string_buffer(int(need))
        lib.ref_rqc_circuit_text(rows, cols, depth, seed, buf, need)
        ctext = buf.value.decode()
        zero = (C.c_uint8 * nq)()
        need = lib.ref_rqc_network_text(rows, cols, depth, seed, zero, None, 0)
        nb = C.create_string_buffer(int(need))
        lib.ref_rqc_network_text(rows, cols, depth, seed, zero, nb, need)
        steps = (C.c_int * (4 * 4096))()
        nst = lib.ref_rqc_path(rows, cols, depth, seed, steps, len(steps))
        path = [[steps[2 * i], steps[2 * i + 1]] for i in range(nst)]
        amps = []
        for x in bitstrings_for(nq, 10, seed):
            xb = (C.c_uint8 * nq)(*x)
            row = {"x": x}
            for label, kw in (("BASELINE", dict(force="FP32_REF")), ("AUTO-0", dict()),
                              ("AUTO-0-lowered", dict(size_auto=4, size_tf32=2)),
                              ("FP16TCEC", dict(force="FP16TCEC")),
                              ("TF32TCEC", dict(force="TF32TCEC")),
                              ("FP16TC", dict(force="FP16TC"))):
                cfg = O.make_config(**kw)
                out = (C.c_float * 2)()
                logbuf = C.create_string_buffer(1 << 16)
                rc = lib.ref_rqc_amplitude(rows, cols, depth, seed, xb, C.byref(cfg), out, None,
                                           logbuf, len(logbuf))
                assert rc == 0
                z = np.array([out[0], out[1]], dtype=np.float32)
                row[label] = bits(z).tolist()
                if label == "AUTO-0-lowered" and x == bitstrings_for(nq, 10, seed)[0]:
                    row["log_lowered"] = [ln for ln in logbuf.value.decode().split("\n") if ln]
            tn = (C.c_double * 2)()
            lib.ref_rqc_amplitude_tn_oracle(rows, cols, depth, seed, xb, tn)
            sv = (C.c_double * 2)()
            lib.ref_rqc_amplitude_sv_oracle(rows, cols, depth, seed, xb, sv)
            row["tn_oracle"] = [tn[0], tn[1]]
            row["sv_oracle"] = [sv[0], sv[1]]
            amps.append(row)
        rq.append({"rows": rows, "cols": cols, "depth": depth, "seed": seed,
                   "circuit_text": ctext,
                   "network_text_sha": hashlib.sha256(nb.value).hexdigest(),
                   "path": path, "amplitudes": amps})
    json.dump(rq, open(os.path.join(OUT, "rqc.json"), "w"))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
