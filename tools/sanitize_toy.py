"""The smallest run of every library kernel on the step path, for compute-sanitizer (SURVEY §4
item 5): toy table (BASELINE configs[0]) at D = 1 — synthetic init + grads, two lamb_step calls
(prologue, pass A TMA ring, finalize, pass B TMA ring), the pre-step kernels once, one
per-bucket step and the self-check — then the result against the oracle.

    python tools/sanitize_toy.py
    compute-sanitizer --tool memcheck --kernel-name kre=lamb --error-exitcode 9 python tools/sanitize_toy.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from gpu_common import compare_state, run_gpu, snapshot_w  # noqa: E402


def main():
    wl = W.toy()
    L = run_gpu(wl, steps=2, device=0)
    torch.cuda.synchronize()
    orc = oracle.OracleRun(wl, world_size=1, mode=oracle.PER_RANK)
    orc.step(1)
    orc.step(2)
    worst = compare_state(L, orc, 2)
    spec = [(t.init, t.gexp) for t in wl.tensors]
    L.set_grad_clip(1e-3)                      # pre-step kernels (grad stats, clip finalize/combine)
    L.synth_grads(spec, wl.seed, 1, 3)
    L.step(3)
    L.set_grad_clip(0.0)
    L.step_bucket(0, 4)                         # per-bucket path
    counts = L.self_check()
    torch.cuda.synchronize()
    assert all(v == 0 for v in counts.values()), counts
    L.close()
    print(f"sanitize_toy ok (max rel err w = {worst:.2e})", flush=True)


if __name__ == "__main__":
    main()
