"""bench.py's output contract: stdout carries exactly one JSON line (rank 0), whatever else the run prints.

CPU: the reference arm (`--impl reference`, the oracle on a bounded C4 sample) alone and under
torch.distributed.run with two gloo ranks (rank 0 prints, rank 1 exits 0 without work).
GPU: a one-step C4 run carries the keys the driver reads (roofline, clocks, gpu_launches, e2e-free form).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cmd, timeout=600):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, f"stdout must be one JSON line, got {len(lines)}: {r.stdout[:500]}"
    return json.loads(lines[0])


def check_reference_line(d, n):
    assert d["impl"] == "reference" and d["n_gpus"] == n
    for k in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_one_line():
    d = run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"])
    check_reference_line(d, 1)


def test_reference_arm_two_ranks_one_line():
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--impl", "reference",
             "--gpus", "2", "--steps", "1", "--warmup", "3"])
    check_reference_line(d, 2)


@pytest.mark.gpu
def test_c4_line_keys():
    d = run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu", "--no-c1",
             "--no-verify"])
    assert d["n_gpus"] == 1 and d["unit"] == "TFLOP/s" and d["value"] > 0
    assert "C4" in d["config"]["workload"]
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert d["gpu_launches"] == 3 and set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
