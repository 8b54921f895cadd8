"""bench.py's multi-rank launcher on CPU: `--gpus 2` re-executes under torch.distributed.run (gloo, --stub
step), every rank runs its shard, the gathered checksum equals the unsharded one and rank 0 prints one JSON
line with n_gpus = 2.  The stub step has no method arithmetic; the CUDA step is the
same code path with the evaluator swapped."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return lines[0]


def test_gpus_2_launches_two_ranks_and_merges():
    one = _run("--stub", "--steps", "1")
    two = _run("--gpus", "2", "--stub", "--steps", "1")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["checksum_matches_unsharded"] is True
    assert two["config"]["checksum"] == one["config"]["checksum"]
    assert two["config"]["integers"] == one["config"]["integers"]
