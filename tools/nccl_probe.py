"""NCCL collective bus bandwidth on this box (busBW = (D-1)/D * bytes / t), 1 GiB
bf16 reduce-scatter and all-gather, for context next to the fused passes' NVLink rates.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/nccl_probe.py
"""
import json
import os

import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
D, r = dist.get_world_size(), dist.get_rank()
out = {"D": D}
for dtype, name in ((torch.bfloat16, "bf16"), (torch.float32, "fp32")):
    n = (1 << 30) // torch.tensor([], dtype=dtype).element_size()
    n -= n % D
    full = torch.ones(n, dtype=dtype, device="cuda")
    part = torch.empty(n // D, dtype=dtype, device="cuda")
    for op in ("rs", "ag"):
        def run():
            if op == "rs":
                dist.reduce_scatter_tensor(part, full)
            else:
                dist.all_gather_into_tensor(full, part)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        out[f"{op}_{name}_ms"] = ms
        out[f"{op}_{name}_busbw_GBps"] = (D - 1) / D * (1 << 30) / (ms * 1e-3) / 1e9
if r == 0:
    print(json.dumps(out))
dist.destroy_process_group()
