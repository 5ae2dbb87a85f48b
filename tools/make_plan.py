"""Precompute a sliced contraction plan (hyper_path) for a Sycamore-class
circuit and store it as JSON (path + sliced labels + a hash of the network
labels), so bench.py need not repeat the CPU search.

    python tools/make_plan.py --cycles 12 --trials 6 --max-log2 28
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.paths import hyper_path  # noqa: E402


def spec_hash(spec):
    h = hashlib.sha256()
    for ls, ds in zip(spec.labels, spec.dims):
        h.update((",".join(ls) + "|" + ",".join(map(str, ds)) + ";").encode())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--cycles", type=int, default=12)
    p.add_argument("--trials", type=int, default=6)
    p.add_argument("--max-log2", type=float, default=28.0)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--time-model", action="store_true")
    p.add_argument("--k", type=int, default=12)
    p.add_argument("--out", default="")
    a = p.parse_args()
    circ = sycamore_like(a.cycles, 1)
    spec = circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])
    t0 = time.time()
    path, sliced, flops, width = hyper_path(spec, a.max_log2, trials=a.trials, seed=a.seed,
                                            log=lambda s: print(s, flush=True),
                                            time_model=a.time_model, k=a.k)
    out = {"circuit": f"sycamore_like({a.cycles}, 1)", "spec_hash": spec_hash(spec),
           "max_log2": a.max_log2, "sliced": sliced, "total_flops": flops, "width_log2": width,
           "search_s": round(time.time() - t0, 1), "time_model": a.time_model, "path": path}
    fn = a.out or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "paper_2303_08989_b200", "plans", f"sycamore_m{a.cycles}.json")
    json.dump(out, open(fn, "w"))
    print(fn, len(path), "steps", len(sliced), "sliced", f"{flops:.3g}", "flops", width)
