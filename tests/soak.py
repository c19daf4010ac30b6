"""Soak test: many consecutive LAMB steps through the C-ABI (test infrastructure: it calls
oracle/, so it lives under tests/).  Checks that the step time does not drift (§6.3
P:991 reports MFU decaying over a long run from skewed collective launches) and that after
many steps the small tensors still match the oracle (barrier epochs, events, graph replay and
the bias-correction constants stay consistent).

    python tests/soak.py --steps 2000 [--graph]
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/soak.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from gpu_common import compare_state, spec_of  # noqa: E402
from paper_2402_15627_b200 import lamb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2000)
ap.add_argument("--chunk", type=int, default=100)
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
pg = None
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pg = dist.group.WORLD

# 1.3B layout for timing; the 1-D tensors (cheap for the oracle) are checked at the end
wl = W.gpt_1p3b()
spec = spec_of(wl)
L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, world_size=world, rank=rank, device=local,
              pg=pg, graph=a.graph)
L.synth_init(spec, wl.seed)
L.synth_grads(spec, wl.seed, rank + 1, 1)   # the same gradients every step (generator step 1)
times = []
s = torch.cuda.current_stream()
t = 0
while t < a.steps:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.chunk):
        t += 1
        L.step(t)
    e1.record(s)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / a.chunk)
ids = [i for i, ts in enumerate(wl.tensors) if ts.numel <= 8192][:40]
orc = oracle.OracleRun(wl, world_size=world, mode=oracle.PER_RANK, tensor_ids=ids)
orc.grads_cache = {i: orc.grads(i, 1) for i in ids}
orc.grads = lambda i, step: orc.grads_cache[i]
for k in range(1, a.steps + 1):
    orc.step(k)
worst = compare_state(L, orc, a.steps, ids=ids, check_params=False)
L.close()
if rank == 0:
    print(json.dumps({"steps": a.steps, "world": world, "graph": a.graph,
                      "ms_per_step_by_chunk": [round(x, 4) for x in times],
                      "drift_last_vs_first": times[-1] / times[0] - 1.0,
                      "parity_after_steps": "ok", "max_rel_err_w": worst}))
if world > 1:
    dist.destroy_process_group()
