"""Multi-GPU parity (FUSED peer-memory path, the NCCL baseline and the NVLS multicast mode),
launched with torchrun, one process per GPU.  Skips when fewer than 2 GPUs are visible."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
needs2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")


def _torchrun(n, *args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tests", "dist_gpu_parity.py"),
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0


@needs2
@pytest.mark.parametrize("mode", ["fused", "nccl"])
def test_parity_2gpu(mode):
    _torchrun(2, "--mode", mode)


@needs2
def test_parity_2gpu_nvls():
    """NVLS mode: reduce-scatter by multimem.ld_reduce, all-gather by
    multimem.st, against the variant oracle g = grad_scale * bf16_rne(sum_j G_j) (reading Z23)."""
    _torchrun(2, "--mode", "nvls")


@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs")
def test_parity_4gpu_nvls():
    _torchrun(4, "--mode", "nvls")


@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("mode", ["fused", "nccl"])
def test_parity_4gpu(mode):
    _torchrun(4, "--mode", mode, *(["--big"] if mode == "fused" else []))


@pytest.mark.skipif(NGPU < 3, reason="needs >= 3 GPUs")
def test_parity_3gpu_fused():
    """Non-power-of-two world: Q = 128 lcm(3, 8) changes the layout, grad_scale = 1/3 is inexact."""
    _torchrun(3, "--mode", "fused")


@pytest.mark.skipif(NGPU < 8, reason="needs 8 GPUs")
def test_parity_8gpu_fused():
    _torchrun(8, "--mode", "fused", "--big")


@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs")
def test_full_size_530b_stress_13b_175b_4gpu():
    """BASELINE configs[2], [3] and [4] at full size on 4 GPUs (141 / 90 / 152 GB per GPU):
    every stress / LayerNorm tensor of the 530B slice, sampled 13B tensors, and every vector
    plus one 603M-element matrix of the 175B slice against the oracle."""
    _torchrun(4, "--mode", "fused", "--full", timeout=1800)


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
def test_parity_8ranks_oversubscribed():
    """D = 8 FUSED on whatever GPUs the box has (ranks share devices, time-sliced): the NS = ND = 8
    kernels, the 8-rank barrier/straddler protocol and the FUSED checkpoint reload, bootstrapped
    without NCCL through lamb_create_with_allgather over a gloo group."""
    _torchrun(8, "--mode", "fused", "--oversub", timeout=1200)


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
@pytest.mark.parametrize("world", [5, 6, 7])
def test_parity_odd_worlds_oversubscribed(world):
    """D = 5, 6, 7 (the NS = ND = 5..7 pass kernels, Q = 128 lcm(D, 8) layouts, inexact
    grad_scale = 1/D) on whatever GPUs the box has, against the oracle: toy, 10 steps, ragged,
    stress straddlers and H8 (replicated gradients == the unsharded D = 1 oracle)."""
    _torchrun(world, "--mode", "fused", "--oversub", "--quick", timeout=900)
