"""bench.py output contract (one JSON line with the keys the driver reads).

CPU: the reference arm (`--impl reference`, the CPU tracker on the host cores).
GPU: our arm on a short run, including roofline, e2e, clocks and the
critical-path model.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5",
                  "--workload", "cyclic16")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_batch_contract():
    """The default workload (C5 batch) on the reference arm: a thread pool over paths."""
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-paths", "8")
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["workload"].startswith("batch8192") and "pool" in d["cpu_baseline"]["sample"]


@pytest.mark.gpu
def test_our_arm_batch_contract(gpu):
    d = run_bench("--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--paths-per-step", "512")
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("batch8192") and d["paths"]["tracked"] == 1024
    assert d["gpu_launches"] == 2 and 0 < d["roofline"]["frac"] < 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 512 * 2 * 2 * 32 * 8


@pytest.mark.gpu
def test_our_arm_contract(gpu):
    d = run_bench("--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--workload", "chandra64")
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["workload"] == "chandra64-dd"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys() and 0 < r["frac"] < 1
    # achieved = the algorithmic work of ONE launch (one tracked path) over the launch time
    per_launch = r["work_per_launch_fp64_instr"] / (d["ms_per_step"] * 1e-3) / 1e12
    assert abs(r["achieved"] - per_launch) <= 0.05 * per_launch, (r["achieved"], per_launch)
    assert r["work_per_launch_fp64_instr"] > d["path"]["newton_iters"] * r["work_per_eval"]
    assert d["gpu_launches"] == 2
    assert d["path"]["success"]
    assert d["critical_path"]["columns_per_solve"] == 64
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
