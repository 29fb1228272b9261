"""bench.py's multi-GPU path, end to end: `--gpus 2` outside torchrun re-launches itself with
torch.distributed.run (2 ranks), each rank takes its slice of the workload's units
(shard.unit_shard) and rank 0 prints ONE line with the whole-job value (strong scaling).  On a
one-GPU box the ranks share cuda:0 with gloo plumbing (`--oversubscribe`: they never wait on each
other's kernels, only on host barriers); the line says so."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_strong_scaling_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--oversubscribe", "--config", "cfgM",
           "--seq-len", "1024", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["units_per_gpu"] == 4
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and "oversubscribed" in d
    assert d["config"]["units"] == 8 and d["gpu_launches"] > 0
