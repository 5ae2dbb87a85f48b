"""bench.py's N > 1 path end to end on the one-GPU test box: `--gpus 2`
re-executes under torch.distributed.run, both ranks share cuda:0 with gloo
(TCEC_BENCH_SHARED_GPU=1; NCCL refuses two ranks on one GPU), the CGEMM runs
as replicas and the sliced Sycamore-class amplitude is sharded over the two
ranks -- and equals the one-rank amplitude bit for bit (slice-ordered f64
sum after one all_gather)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(gpus):
    env = dict(os.environ, TCEC_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--n", "2048",
           "--steps", "2", "--warmup", "3", "--no-sweep", "--no-cpu", "--no-legs", "--no-pageable",
           "--sliced-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_match_one_rank():
    one = _run(1)
    two = _run(2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert "over 2 GPU(s)" in two["sliced_rcs"]["config"]["workload"]
    assert two["sliced_rcs"]["amplitude"] == one["sliced_rcs"]["amplitude"]
    assert two["config"]["decision"] == one["config"]["decision"]
