"""Precompute a sliced contraction plan (paths.hyper_path) for a
Sycamore-class circuit and store it as JSON (path + sliced labels + a hash of
the network labels), so bench.py need not repeat the CPU search.  Trials run
in parallel processes; the plan with the least modelled B200 time wins.

    python tools/make_plan.py --cycles 12 --trials 32 --jobs 8 --time-model --k 14
"""
import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08989_b200.circuits import circuit_to_network, sycamore_like  # noqa: E402
from paper_2303_08989_b200.paths import hyper_path, path_model_cost  # noqa: E402


def spec_hash(spec):
    h = hashlib.sha256()
    for ls, ds in zip(spec.labels, spec.dims):
        h.update((",".join(ls) + "|" + ",".join(map(str, ds)) + ";").encode())
    return h.hexdigest()[:16]


def _spec(cycles):
    circ = sycamore_like(cycles, 1)
    return circuit_to_network(circ, [(q * 7 + 3) % 2 for q in range(circ.n_qubits)])


def _trial(args):
    cycles, max_log2, seed, time_model, k = args
    spec = _spec(cycles)
    path, sliced, flops, width = hyper_path(spec, max_log2, trials=1, seed=seed,
                                            time_model=time_model, k=k)
    return seed, path, sliced, flops, width, path_model_cost(spec, path, sliced, True)


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--cycles", type=int, default=12)
    p.add_argument("--trials", type=int, default=6)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--max-log2", type=float, default=28.0)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--time-model", action="store_true")
    p.add_argument("--k", type=int, default=12)
    p.add_argument("--out", default="")
    a = p.parse_args()
    spec = _spec(a.cycles)
    t0 = time.time()
    jobs = [(a.cycles, a.max_log2, a.seed + 1000 * t, a.time_model, a.k) for t in range(a.trials)]
    best = None
    with mp.Pool(max(1, a.jobs)) as pool:
        for seed, path, sliced, flops, width, model in pool.imap_unordered(_trial, jobs):
            print(f"seed {seed}: {len(sliced)} sliced, 2^{width:.0f}, {flops:.3g} flops, "
                  f"model time {model:.3g}", flush=True)
            if best is None or model < best[5]:
                best = (seed, path, sliced, flops, width, model)
    seed, path, sliced, flops, width, model = best
    out = {"circuit": f"sycamore_like({a.cycles}, 1)", "spec_hash": spec_hash(spec),
           "max_log2": a.max_log2, "sliced": sliced, "total_flops": flops, "width_log2": width,
           "model_time": model, "seed": seed, "search_s": round(time.time() - t0, 1),
           "time_model": a.time_model, "k": a.k, "path": path}
    fn = a.out or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "paper_2303_08989_b200", "plans", f"sycamore_m{a.cycles}.json")
    json.dump(out, open(fn, "w"))
    print(fn, len(path), "steps", len(sliced), "sliced", f"{flops:.3g}", "flops", width, f"model {model:.3g}")
