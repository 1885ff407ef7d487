"""bench.py keeps the driver's JSON contract (one line, required keys, sane values)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
            "gpu_launches", "roofline", "clocks"]


def _run(args):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_has_contract_keys():
    d = _run(["--config", "0", "--steps", "1", "--warmup", "3", "--cpu-budget", "2"])
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"] and d["config"]["all_converged"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_slab_line():
    d = _run(["--config", "4", "--steps", "1", "--warmup", "3", "--no-cpu", "--slabs-per-gpu", "2"])
    assert d["scaling"] == "strong" and d["config"]["slabs"] == 2
    assert d["config"]["all_converged"] and d["value"] > 0
