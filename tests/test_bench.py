"""bench.py driver contract on CPU: the --gpus N self-launch (torchrun with N
gloo ranks in --plan-only mode), the per-rank layer plan of the sharded
config 5, the default configurations, and the reference arm's line.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BENCH = ROOT / "bench.py"


def _run(*argv, timeout=300):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    r = subprocess.run([sys.executable, str(BENCH), *argv], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", BENCH)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_default_config_single_gpu_is_vgg16():
    d = _run("--plan-only")
    assert d["n_gpus"] == 1
    assert d["config"]["workload"].startswith("BASELINE config 4")
    assert len(d["config"]["layers"]) == 13
    assert all(p["shard"] == "replica" and p["n"] == 64 for p in d["ranks"][0]["plan"])


def test_gpus2_relaunches_two_ranks_with_config5_shards():
    d = _run("--gpus", "2", "--plan-only")
    assert d["n_gpus"] == 2
    assert d["config"]["workload"].startswith("BASELINE config 5")
    assert d["config"]["parallelism"] == "batch-shard2+cout-shard2"
    ranks = sorted(d["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == [0, 1]
    for r in ranks:
        by = {p["name"]: p for p in r["plan"]}
        # batch shards: samples [N r/P, N (r+1)/P) of the N=256 layers
        for name in ("conv1x1_64to256@56_n256", "conv128@28_n256", "conv256@14_n256"):
            assert by[name]["shard"] == "batch" and by[name]["n"] == 128
        # c_o shard of 512@7 N=8: the whole batch, half the output channels
        co = by["conv512@7_n8_coshard"]
        assert co["shard"] == "cout" and co["n"] == 8
        assert (co["c_lo"], co["c_hi"]) == ((0, 256) if r["rank"] == 0 else (256, 512))
    # distinct seeds per rank for the batch shards (different samples)
    s0 = {p["name"]: p["seed"] for p in ranks[0]["plan"]}
    s1 = {p["name"]: p["seed"] for p in ranks[1]["plan"]}
    assert s0["conv128@28_n256"] != s1["conv128@28_n256"]
    assert s0["conv512@7_n8_coshard"] == s1["conv512@7_n8_coshard"]


def test_gpus3_uneven_cout_partition():
    d = _run("--gpus", "3", "--plan-only", "--config", "5")
    ranks = sorted(d["ranks"], key=lambda r: r["rank"])
    cuts = [(p["c_lo"], p["c_hi"]) for r in ranks for p in r["plan"] if p["shard"] == "cout"]
    assert cuts[0][0] == 0 and cuts[-1][1] == 512
    assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
    assert sum(p["n"] for r in ranks for p in r["plan"] if p["name"] == "conv128@28_n256") == 256


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(BENCH), "--gpus", "1", "--plan-only"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=str(ROOT))
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_both_arms_share_the_config_dict():
    bench = _bench_module()

    class A:
        config = 2
        replicas = 0
        steps = 20
    for world in (1, 2):
        c = bench.workload_config(A, world)
        assert set(c) == {"workload", "layers", "batch", "parallelism", "l2"}


def test_reference_arm_line_config1():
    d = _run("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1", timeout=600)
    assert d["impl"] == "reference"
    assert d["unit"] == "GFLOP/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["cpu_model"]
    assert cb["kind"] in ("reference", "port")
    bench = _bench_module()

    class A:
        config = 1
        replicas = 0
        steps = 1
    assert d["config"] == bench.workload_config(A, 1)


@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "smmconv").exists(),
                    reason="reference not installed under baseline/_ref")
def test_reference_sample_matches_oracle_bitwise():
    """The reference arm's compute is the reference itself: its output on a
    small layer equals the C restatement bitwise."""
    import numpy as np

    from oracle import smm_oracle as orc
    from paper_2411_15659_b200 import ConvGeometry, repack_weights
    bench = _bench_module()
    g = ConvGeometry(4, 6, 9, 8, 3, 3, 1, 1, 1, 1)
    plan = [dict(name="t", n=1, g=g, seed=5, shard="replica", c_lo=0, c_hi=6)]
    ref = bench.ReferenceSample(plan, 2)
    assert ref.kind == "reference"
    y = ref.run()[0]
    x, w = ref.items[0][1], ref.items[0][0].weights
    y2 = orc.smm_conv_c(x[0], repack_weights(np.asarray(w, np.float32), g), g, threads=1)
    assert np.array_equal(y, y2)
