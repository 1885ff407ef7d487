"""bench.py's own multi-rank flow on CPU: `--gpus 2` with no launcher spawns two ranks
(RANK/WORLD_SIZE, rendezvous on 127.0.0.1) that run run_b200's orchestration with gloo
(--dry-run: sharding, barrier-bracketed timing, max over ranks, report gathering) and
rank 0 prints one JSON line with n_gpus = 2."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*extra):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "2", "--warmup", "3", *extra], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_weak_scaling_two_ranks():
    d = _run("--batch", "5")
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["global_batch"] == 10 and d["config"]["batch_per_gpu"] == 5
    assert d["report_order"] == list(range(10))
    # every rank drew its own batch (seed 2000 + rank)
    a, b = (np.asarray(m) for m in d["mus_by_rank"])
    assert a.shape == b.shape == (5, 4) and not np.array_equal(a, b)
    # whole-job rate from the slowest rank: 10 solves per step
    assert d["value"] == pytest.approx(10 / (d["ms_per_step"] / 1e3), rel=1e-2)


def test_strong_scaling_shards_one_global_batch():
    from paper_2311_13862_b200.problems import sample_mus, thermal_block
    d = _run("--batch", "7", "--scaling", "strong")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 7
    got = np.concatenate([np.asarray(m) for m in d["mus_by_rank"]])
    np.testing.assert_array_equal(got, sample_mus(thermal_block((2, 2, 1)), 7, seed=2000))
    assert [len(m) for m in d["mus_by_rank"]] == [4, 3]
    assert d["report_order"] == list(range(7))
