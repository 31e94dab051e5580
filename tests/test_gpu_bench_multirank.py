"""bench.py's N>1 path end to end on the one leased GPU: `--gpus 2`
self-launches two torchrun ranks; with SMMC_BENCH_BACKEND=gloo both share
cuda:0 (NCCL refuses two ranks per device), so the sharded config-5 step --
batch shards, the c_o-shard layer's fused peer-write gather over CUDA IPC
with its fences, the max-over-ranks timing and rank 0's JSON line -- runs
for real.  A plumbing check: the timings of two ranks on one GPU mean
nothing."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_one_gpu_gloo():
    env = dict(os.environ, SMMC_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "1", "--no-cpu-baseline", "--no-e2e"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("BASELINE config 5")
    assert d["config"]["parallelism"] == "batch-shard2+cout-shard2"
    assert d["gather_path"].startswith("fused peer-write")
    assert d["value"] > 0 and d["gpu_launches"] > 0
