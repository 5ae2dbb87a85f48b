"""A/B of an environment toggle on the configs[2] skewed leg: per-shape stage
times (stats / prep / gemm, CUDA events) of `bench.py --workload skewed`, arms
alternated twice, best of the two runs per arm.

    python tools/ab_env_skewed.py TCEC_STATS_KEEP 0 1
"""
import json
import os
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
var, vals = sys.argv[1], sys.argv[2:]
runs = {v: [] for v in vals}
for _ in range(2):
    for v in vals:
        env = dict(os.environ, **{var: v})
        r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "skewed", "--steps", "20",
                            "--warmup", "3"], env=env, capture_output=True, text=True, cwd=root)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(r.stderr[-2000:])
            sys.exit(1)
        runs[v].append(json.loads(line[-1]))
shapes = runs[vals[0]][0]["shapes"]
for i, s in enumerate(shapes):
    cells = []
    for v in vals:
        best = min(runs[v], key=lambda d: d["shapes"][i]["ms"])["shapes"][i]
        st = best.get("stages_ms", {})
        cells.append(f"{var}={v}: {best['ms'] * 1e3:8.1f} us (stats {st.get('stats', 0) * 1e3:6.1f} "
                     f"prep {st.get('prep', 0) * 1e3:6.1f} gemm {st.get('gemm', 0) * 1e3:7.1f})")
    print(f"({s['m']},{s['n']},{s['k']}) " + " | ".join(cells), flush=True)
for v in vals:
    print(f"{var}={v}: leg value {max(d['value'] for d in runs[v])} TFLOP/s")
