"""bench.py's multi-rank launcher on the CPU: ``--gpus 2`` without a torchrun
environment re-launches itself through torch.distributed.run with two ranks
(127.0.0.1 rendezvous); --dry-run swaps the GPU work for a gloo reduction, so
the rank set-up, the world-size check and the one-line rank-0 output are what
is exercised."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra, env=None):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *extra],
                          capture_output=True, text=True, timeout=300, env=e, cwd=ROOT)


def test_two_rank_relaunch_prints_one_line():
    r = _run("--gpus", "2", "--steps", "3", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["max_over_ranks"] == 2.0  # rank 1's value won the max
    assert line["config"]["global_batch"] == 2 * line["config"]["fields_per_gpu"]


def test_single_rank_default():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["n_gpus"] == 1 and line["max_over_ranks"] == 1.0


def test_world_size_mismatch_is_refused():
    r = _run("--gpus", "2", env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
