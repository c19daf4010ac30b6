"""Measure the two-stage checkpoint (NEXT #4) on one GPU: stage 1 (device -> pinned host,
blocking), stage 2 (background file write), and load (file -> device + param rebuild).

    python tools/bench_ckpt.py --config gpt1.3b --path /tmp/lamb.ckpt
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2402_15627_b200 import lamb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt1.3b")
ap.add_argument("--path", default="/tmp/lamb_bench.ckpt")
a = ap.parse_args()
wl = W.get(a.config)
spec = [(t.init, t.gexp) for t in wl.tensors]
L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=wl.cap)
L.synth_init(spec, wl.seed)
L.synth_grads(spec, wl.seed, 1, 1)
L.step(1)
torch.cuda.synchronize()
L.checkpoint_save(a.path, 1)          # first save allocates the pinned staging buffer
L.checkpoint_wait()
state_bytes = 12 * L.plan.shard_size
t0 = time.perf_counter()
L.checkpoint_save(a.path, 1)
t1 = time.perf_counter()
# training continues during stage 2
for t in range(2, 6):
    L.step(t)
torch.cuda.synchronize()
t2 = time.perf_counter()
L.checkpoint_wait()
t3 = time.perf_counter()
L.close()
B = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, bucket_cap=wl.cap)
t4 = time.perf_counter()
B.checkpoint_load(a.path)
t5 = time.perf_counter()
B.close()
os.remove(a.path)
print(json.dumps({"config": wl.name, "state_bytes": state_bytes,
                  "stage1_s": t1 - t0, "stage1_GBps": state_bytes / (t1 - t0) / 1e9,
                  "stage2_s_total": t3 - t0, "steps_during_stage2": 4,
                  "stage2_GBps": state_bytes / (t3 - t1) / 1e9,
                  "load_s": t5 - t4, "load_GBps": state_bytes / (t5 - t4) / 1e9}))
