"""L2 reuse between pass A and pass B at the bucket level (D = 1): a table of T equal tensors of S
elements, one per bucket (cap = S), stepped (a) whole (pass A over everything, then pass B)
and (b) bucket by bucket (pass A / finalize / pass B of bucket b before bucket b+1), where
pass B can find bucket b's m, v, w still in L2.  CUDA events, median of 10 steps.

    python tools/l2_bucket_probe.py  -> one JSON line per S
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2402_15627_b200 import lamb  # noqa: E402

TOTAL = 1 << 30
for S in (2 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20):
    T = TOTAL // S
    tensors = [W.TensorSpec(f"t{i}", S, W.DECAY, W.INIT_UNIFORM, W.GEXP_MATRIX) for i in range(T)]
    wl = W.Workload(f"eq{S}", 90, tensors, W.default_groups(), S)
    spec = [(t.init, t.gexp) for t in tensors]
    L = lamb.Lamb([(t.numel, t.group) for t in tensors], wl.groups, bucket_cap=S)
    L.synth_init(spec, wl.seed)
    L.synth_grads(spec, wl.seed, 1, 1)
    nb = L.plan.buckets.shape[0]
    res = {"S_M": S >> 20, "tensors": T, "buckets": nb}
    for mode in ("whole", "bucket", "whole", "bucket"):
        times = []
        for t in range(1, 13):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if mode == "whole":
                L.step(t)
            else:
                for b in range(nb):
                    L.step_bucket(b, t)
            e1.record()
            torch.cuda.synchronize()
            if t > 2:
                times.append(e0.elapsed_time(e1))
        res[mode] = round(float(np.median(times)), 4)
    L.close()
    print(json.dumps(res), flush=True)
