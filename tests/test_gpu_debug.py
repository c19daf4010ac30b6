"""The LAMB_DEBUG build (liblamb_debug.so) on the GPU — the substitute for compute-sanitizer,
which is closed on this pool: its device-side checks (item bounds and
alignment, ring-stage tags, bounded mbarrier waits, segment / straddler / barrier-epoch bounds)
stay silent on the parity workloads, including the 8-rank protocol, and DO fire when an item
table is corrupted on purpose (lamb_debug_corrupt_item): a "LAMB_DEBUG" message and a trap
instead of an out-of-bounds access."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]
ENV = dict(os.environ, LAMB_DEBUG_LIB="1")

CORRUPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
import torch, workloads as W
from paper_2402_15627_b200 import lamb
from gpu_common import run_gpu
assert lamb.DEBUG and lamb.LIB_PATH.endswith("liblamb_debug.so")
wl = W.toy()
L = run_gpu(wl, steps=1)
torch.cuda.synchronize()
print("step 1 ok", flush=True)
n = L.plan.flat_size
lamb.check(lamb.lamb_debug_corrupt_item(L.h, 1, {flat_off}), L.h)
L.step(2)
torch.cuda.synchronize()
print("NOT DETECTED", flush=True)
"""


def _run(code):
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT,
                          env=ENV)


@pytest.mark.parametrize("flat_off,what", [(12, "not 8-aligned"), (1 << 40, "flat range")])
def test_debug_checks_fire_on_a_corrupted_item(flat_off, what):
    r = _run(CORRUPT.format(root=ROOT, flat_off=flat_off))
    out = r.stdout + r.stderr
    assert "step 1 ok" in out, out[-2000:]
    assert "NOT DETECTED" not in out and r.returncode != 0, out[-2000:]
    assert "LAMB_DEBUG" in out and what in out, out[-2000:]


def test_debug_build_silent_on_the_parity_suite():
    # single-GPU parity cases (toy at both lrs, ragged tables, group variants, stress-like,
    # determinism, per-bucket stepping, CUDA graph, host pipeline) on the debug library
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-s", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "toy_parity or ragged or group_variants or determinism or step_bucket or graph or "
                        "step_host_pipeline or zero_grad"],
                       capture_output=True, text=True, timeout=1500, cwd=ROOT, env=ENV)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "LAMB_DEBUG" not in r.stdout + r.stderr, (r.stdout + r.stderr)[-3000:]
    assert "liblamb_debug.so" in r.stdout and " passed" in r.stdout


def test_debug_build_silent_on_8_ranks_oversubscribed():
    # the D = 8 kernels (8 gradient sources, 8 param destinations), barriers, straddler
    # exchange, checkpoint reshard, pre-step, copy-engine schedule — every check on
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "dist_gpu_parity.py"),
           "--mode", "fused", "--oversub"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=ENV)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "LAMB_DEBUG" not in r.stdout + r.stderr, (r.stdout + r.stderr)[-3000:]
    assert "liblamb_debug.so" in r.stdout and "[ok] toy D=8" in r.stdout
