"""CPU check of bench.py's contract: the reference arm (the CPU oracle on a bounded sample)
prints ONE JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "params/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "gpt1.3b"


def test_reference_arm_other_ranks_exit_quietly():
    # under torchrun (N > 1) rank 0 alone runs the oracle and prints; the others exit 0 without work
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_reference_arm_config_is_our_arms_config():
    # the driver compares the two arms' `config`: the reference line carries our arm's config for
    # the same arguments (flat_size from the oracle planner == the library planner's, H12)
    sys.path.insert(0, ROOT)
    import bench
    import workloads as W
    from paper_2402_15627_b200 import lamb
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    wl = W.get("gpt1.3b")
    pv = lamb.host_plan([t.numel for t in wl.tensors], 1, 0, wl.cap)
    ours = bench.run_config(bench.parse([]), wl, 1, int(pv.flat_size))
    assert ref["config"] == ours
