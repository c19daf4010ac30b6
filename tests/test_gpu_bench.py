"""GPU check of bench.py's JSON contract on our arm (short runs)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run("--steps", "3", "--warmup", "3", "--cpu-seconds", "2", "--curve-steps", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "gpt1.3b"
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["unit"] == "GB/s" and r["traffic"] > 0
    assert d["gpu_launches"] >= 3 * 3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["ranks_seen"] == 1
    c = d["cpu_baseline"]   # SURVEY §8(d) oracle timing: all cores and 1 core, toy full step, labelled extrapolation
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] >= 1 and c["cores_1core"] == 1
    assert c["toy_full_step_ms"] > 0 and c["extrapolated"] is True and c["full_step_ms"] > 0
    nc = d["north_star_curve"]   # the north star's scaling-curve layout, timed the same way
    assert nc["workload"] == "175b_slice_3l" and nc["value"] > 0 and 0 < nc["roofline"]["frac"] < 1.2


def test_bench_self_launch_two_ranks():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    d = run("--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-curve")
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2 and d["config"]["parallelism"] == "zero2-dp2"
    assert "nvlink" in d["roofline"] and d["roofline"]["nvlink"]["bytes_in_per_gpu"] > 0


def test_bench_small_config_and_graph():
    d = run("--config", "toy", "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--graph")
    assert d["north_star_curve"] is None   # not timed with --graph
    assert d["config"]["workload"] == "toy" and d["config"]["cuda_graph"] and d["value"] > 0
