"""bench.py's CPU-side contract at tiny sizes: the reference arm prints one JSON line carrying
the contract keys (metric/value/unit/steps/warmup/ms_per_step/config/e2e/cpu_baseline, impl =
reference) and rank > 0 of a torchrun launch exits without output; `--gpus 2 --dry-run`
launches two gloo ranks itself and reports n_gpus 2 with config 3's global batch unchanged;
the batch x KV-head shard plan covers every lane exactly once."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(extra_env=None):
    env = dict(os.environ, **(extra_env or {}))
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--ctx", "2048", "--steps", "1",
           "--warmup", "1", "--cpu-lanes", "2", "--cpu-steps", "1", "--layers", "4"]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    assert d["config"]["workload"].startswith("llama7b-attn-2k")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "lanes x 1 steps" in cb["sample"]


def test_reference_arm_nonzero_rank_is_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_dry_run_two_ranks_strong_scaling():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--ctx", "1024", "--layers", "2",
           "--steps", "1", "--warmup", "1"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 8 and d["lanes_total"] == 8 * 32
    assert d["config"]["workload"] == "llama7b-attn-1k-b8-int4-planted"


def test_shard_plan_covers_lanes():
    sys.path.insert(0, str(ROOT))
    import bench
    for B, H, Hkv in ((8, 32, 32), (8, 32, 8), (1, 32, 32), (16, 32, 8)):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                sp = bench.shard_plan(B, H, Hkv, world, r)
                assert sp["global_batch"] == B and sp["q_lanes"] == sp["kv_lanes"] * (H // Hkv)
                seen += list(range(sp["kv0"], sp["kv0"] + sp["kv_lanes"]))
                assert sp["q0"] == sp["kv0"] * (H // Hkv)
            assert seen == list(range(B * Hkv))
    w = [bench.shard_plan(8, 32, 32, 4, r, "weak") for r in range(4)]
    assert all(x["global_batch"] == 32 and x["kv_lanes"] == 8 * 32 for x in w)
