"""bench.py's reference arm on CPU (no GPU needed): the contract's JSON
line with impl=reference, the workload's metric/unit, a cpu_baseline that
describes the run, and an e2e object carrying the same value."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "distgcn")),
                    reason="baseline/_ref (the reference install) is absent")
def test_reference_arm_line_rmat14():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "rmat14", "--steps", "1", "--warmup", "1",
                        "--ref-budget", "0.5"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "gcn_epoch_ms" and line["unit"] == "ms"
    assert line["higher_is_better"] is False
    assert line["value"] > 0 and line["ms_per_step"] == line["value"]
    cb = line["cpu_baseline"]
    # the unchanged reference (baseline/_ref) at config 1's p=4 ranks, timed in full
    assert cb["kind"] == "reference" and cb["cores"] == 4 and cb["value"] == line["value"]
    assert line["value_kind"].startswith("measured")
    assert line["e2e"] == {"value": line["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "R-MAT" in line["config"]["workload"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "rmat14", "--gpus", "2"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""
