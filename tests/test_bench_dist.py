"""bench.py's multi-rank plumbing on CPU: `bench.py --gpus 2` re-launches
itself under torch.distributed.run with two ranks (gloo in the
--plumbing-only mode), each rank reduces its contiguous shard, and rank 0
reports n_gpus 2 and the merged best -- equal to the single-rank argmin of
the same synthetic costs."""
from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(gpus, n):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
              "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
         "--n", str(n), "--plumbing-only"], capture_output=True, text=True,
        env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_two_ranks_merge_equals_one_rank():
    n = 1_000_003
    one = _run(1, n)
    two = _run(2, n)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["best"] == one["best"]
    assert one["best"]["index"] >= 0
