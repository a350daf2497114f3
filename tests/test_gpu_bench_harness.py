"""bench.py's multi-rank harness (the --gpus N path the driver's scaling run
uses) on the one GPU available: `--gpus 2 --dist-backend gloo` self-launches 2
ranks with torch.distributed.run, both on cuda:0, each scanning its shard of
C3 through the product RSS path (dist.sharded_exclusive), the totals exchanged
through host memory.  The numbers are not comparable (two ranks share one
GPU); what is checked is the line: n_gpus, shard parallelism, the per-phase
breakdown (max over ranks) and the roofline of the shard-scan kernel."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--config", "C3", "--steps", "3", "--warmup", "3", "--no-e2e"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("shard2")
    assert set(d["phases_ms"]) == {"shard_reduce", "all_gather", "carry", "shard_scan"}
    assert all(v > 0 for v in d["phases_ms"].values())
    assert d["roofline"]["achieved"] > 0 and d["gpu_launches"] >= 3 * 3
