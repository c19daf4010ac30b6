"""Minimal driver for ncu captures: create a handle for a workload, run `--steps` LAMB steps
through the C-ABI (synthetic inputs).  Usage under ncu: see profiles/README.md."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2402_15627_b200 import lamb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt1.3b")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--layers", type=int, default=0, help="truncate a gpt config to this many layers")
a = ap.parse_args()
wl = W.get(a.config)
if a.layers:
    h = {"gpt1.3b": 2048, "gpt13b": 5120}[a.config]
    wl = W.Workload(wl.name + f"-{a.layers}l", wl.index, W.gpt(h, a.layers), wl.groups, wl.cap)
spec = [(t.init, t.gexp) for t in wl.tensors]
L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=wl.cap)
L.synth_init(spec, wl.seed)
L.synth_grads(spec, wl.seed, 1, 1)
for t in range(1, a.steps + 1):
    L.step(t)
torch.cuda.synchronize()
print("ok", wl.name, wl.n_params, "launches", L.launch_count())
L.close()
