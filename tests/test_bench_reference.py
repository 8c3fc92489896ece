"""The reference (CPU) arm of bench.py on this host: one JSON line with the contract's keys,
for a single-matrix config and for the multi-GPU config's bounded row sample (C5 at a
reduced R-MAT scale)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _check(d, workload):
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["config"]["workload"] == workload and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_c1():
    _check(_run(["--workload", "C1", "--steps", "2", "--warmup", "1"]), "C1")


def test_reference_arm_uses_every_core_under_a_launcher(monkeypatch):
    """torchrun exports OMP_NUM_THREADS=1 to each rank; the CPU arm (rank 0 only) must still
    run on all the cores it may use."""
    monkeypatch.setenv("OMP_NUM_THREADS", "1")
    d = _run(["--workload", "C1", "--steps", "1", "--warmup", "1"])
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


@pytest.mark.parametrize("share", ["4", "16"])
def test_reference_arm_c5_row_sample(share, monkeypatch):
    monkeypatch.setenv("KP_REF_C5_SAMPLE", share)
    d = _run(["--workload", "C5", "--scale", "14", "--steps", "1", "--warmup", "1", "--iters", "2"])
    _check(d, "C5")
    smp = d["config"]["sample"]
    assert 0 < smp["nnz"] <= d["config"]["nnz"] and 0 < smp["rows"] <= d["config"]["rows"]
    assert abs(smp["share_of_nnz"] - 1 / int(share)) < 0.05
    assert d["scaling"] == "strong" and d["config"]["iterations"] == 2
