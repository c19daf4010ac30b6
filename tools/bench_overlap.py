"""NEXT #2 measurement: overlap of the sharded LAMB step with a synthetic forward/backward, the
paper's DP overlap (§3.2: RS of a chunk right after its backward, AG right
before its forward, the first AG prefetched, priority = order of the dependent compute).

The forward/backward is a synthetic compute load: per bucket b, bf16 GEMMs (cuBLAS via torch,
a plain library GEMM standing in for the model) worth 2*P_b*tokens FLOPs forward and twice that
backward.  Three iteration schedules, timed with CUDA events on the compute stream, max over
ranks:
  compute  - forward + backward only (the floor),
  serial   - forward + backward, then lamb_step (RS + update + AG exposed),
  overlap  - per bucket: lamb_step_bucket(b, defer AG) on a second stream as soon as b's
             backward is done; lamb_gather_bucket(b) before b's next forward (prefetched in
             bucket order at the start of the iteration).
  ce       - the copy-engine schedule (D > 1): lamb_push_grads_bucket(b) right after b's
             backward (the reduce-scatter traffic on the DMA engines, no SMs), lamb_step_staged
             after the backward (local-HBM update, then the all-gather pushes on the DMA
             engines), lamb_wait_params_bucket(b) before b's next forward.
    python tools/bench_overlap.py --config gpt1.3b --tokens 4096
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/bench_overlap.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads as W  # noqa: E402
from paper_2402_15627_b200 import lamb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt1.3b")
ap.add_argument("--tokens", type=int, default=4096, help="tokens per GPU per iteration")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--ctas", default="0,74,37", help="SM budgets (max CTAs) to try in overlap mode")
ap.add_argument("--green", default="16,32,48",
                help="green-context SM partitions to try (LAMB gets these SMs, the GEMMs the rest)")
ap.add_argument("--carveouts", default="",
                help="cuBLAS SM carve-outs to try (LAMB gets max_ctas = 2 x carve-out)")
ap.add_argument("--cap", type=int, default=0, help="bucket cap (0 = the workload's)")
ap.add_argument("--K", type=int, default=2048, help="synthetic GEMM size [tokens,K]x[K,K]")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
pg = None
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pg = dist.group.WORLD

wl = W.get(a.config)
spec = [(t.init, t.gexp) for t in wl.tensors]
L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, world_size=world, rank=rank,
              device=local, bucket_cap=a.cap or wl.cap, pg=pg, ce=world > 1)
L.synth_init(spec, wl.seed)
L.synth_grads(spec, wl.seed, rank + 1, 1)
B = len(L.plan.buckets)
params_b = [sum(wl.tensors[i].numel for i in range(int(t0), int(t1))) for (_, _, t0, t1) in L.plan.buckets.tolist()]

# synthetic compute: GEMM [tokens, K] x [K, K]
K = a.K
X = torch.randn(a.tokens, K, device="cuda", dtype=torch.bfloat16)
Wm = torch.randn(K, K, device="cuda", dtype=torch.bfloat16)
Y = torch.empty(a.tokens, K, device="cuda", dtype=torch.bfloat16)
gemm_flops = 2.0 * a.tokens * K * K
reps_f = [max(1, round(2.0 * P * a.tokens / gemm_flops)) for P in params_b]


def gemms(n):
    for _ in range(n):
        torch.matmul(X, Wm, out=Y)   # on the current stream (set by iteration)


comp = torch.cuda.current_stream()
ls = torch.cuda.Stream(priority=-1)   # the paper's "high priority communication first"
ev_grad = [torch.cuda.Event() for _ in range(B)]
ev_gath = [torch.cuda.Event() for _ in range(B)]
ev_ls_done = torch.cuda.Event()
step = [0]
last_ce = [0]   # last step done by lamb_step_staged (its params are pushed into the next forward)
ce_events = []  # per "ce" iteration: forward start / backward start / step start / step end


def iteration(mode, comp=comp, ls=ls):
    step[0] += 1
    t = step[0]
    torch.cuda.set_stream(comp)
    if mode == "overlap":
        # forward: gathers issued in bucket order (the first is the prefetch), each forward waits
        with torch.cuda.stream(ls):
            for b in range(B):
                L.gather_bucket(b, stream=ls)
                ev_gath[b].record(ls)
        for b in range(B):
            comp.wait_event(ev_gath[b])
            gemms(reps_f[b])
        for b in reversed(range(B)):
            gemms(2 * reps_f[b])
            ev_grad[b].record(comp)
            ls.wait_event(ev_grad[b])
            L.step_bucket(b, t, defer_ag=True, stream=ls)
        ev_ls_done.record(ls)
        comp.wait_event(ev_ls_done)
    elif mode == "ce":
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(comp)
        for b in range(B):
            if last_ce[0]:
                L.wait_params_bucket(b, last_ce[0], stream=comp)
            gemms(reps_f[b])
        ev[1].record(comp)
        for b in reversed(range(B)):
            gemms(2 * reps_f[b])
            L.push_grads_bucket(b, t, stream=comp)
        ev[2].record(comp)
        L.step_staged(t, stream=comp)
        ev[3].record(comp)
        ce_events.append(ev)
        last_ce[0] = t
    else:
        for b in range(B):
            gemms(reps_f[b])
        for b in reversed(range(B)):
            gemms(2 * reps_f[b])
        if mode == "serial":
            L.step(t, stream=comp)
        elif mode == "serial_buckets":   # per-bucket overhead without any overlap
            for b in reversed(range(B)):
                L.step_bucket(b, t, stream=comp)


def timed(mode, comp=comp, ls=ls):
    for _ in range(a.warmup):
        iteration(mode, comp, ls)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(a.iters):
        iteration(mode, comp, ls)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    if world > 1:
        x = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x)
    return ms


res = {}
for m in ("compute", "serial", "serial_buckets") + (("ce",) if world > 1 else ()):
    res[m] = timed(m)
if world > 1:
    # the first timed "ce" iteration waited on the params of a staged step; re-time after the
    # other modes ran, then the next "ce" run waits on last_ce again (it is still current)
    ce_events.clear()
    res["ce"] = min(res["ce"], timed("ce"))
    torch.cuda.synchronize()
    ph = [[e[i].elapsed_time(e[i + 1]) for i in range(3)] for e in ce_events[a.warmup:]]
    ce_phases = {k: sum(x[i] for x in ph) / len(ph) for i, k in enumerate(("forward", "backward", "step_staged"))}
    # the same phases without any transfer in flight (compute mode) for comparison
    fwd_c = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fwd_c[0].record(comp)
    gemms(sum(reps_f))
    fwd_c[1].record(comp)
    gemms(2 * sum(reps_f))
    fwd_c[2].record(comp)
    torch.cuda.synchronize()
    ce_phases["forward_compute_only"] = fwd_c[0].elapsed_time(fwd_c[1])
    ce_phases["backward_compute_only"] = fwd_c[1].elapsed_time(fwd_c[2])
over = {}
for c in [int(x) for x in a.ctas.split(",")]:
    L.set_max_ctas(c)
    over[c] = timed("overlap")
for k in [int(x) for x in a.carveouts.split(",") if x]:
    # the GEMMs leave k SMs free (cuBLAS SM-count target); the LAMB passes take exactly those
    torch._C._set_sm_carveout_experimental(k)
    L.set_max_ctas(2 * k)
    over[f"carveout{k}"] = timed("overlap")
    res[f"compute_carveout{k}"] = timed("compute")
    torch._C._set_sm_carveout_experimental(0)
torch.cuda.set_stream(comp)
for k in [int(x) for x in a.green.split(",") if x]:
    # hard SM partition: LAMB on k SMs, the GEMMs on the other 148 - k
    lp, cpp, got = lamb.sm_partition(local, k)
    gls, gcs = torch.cuda.ExternalStream(lp), torch.cuda.ExternalStream(cpp)
    L.set_max_ctas(2 * got)
    over[f"green{got}"] = timed("overlap", gcs, gls)
    res[f"compute_green{got}"] = timed("compute", gcs, gls)
    torch.cuda.set_stream(comp)
L.set_max_ctas(0)
res["compute"] = min(res["compute"], timed("compute"))
if rank == 0:
    exposed_serial = res["serial"] - res["compute"]
    best = min(over, key=over.get)
    exposed_overlap = over[best] - res["compute"]
    print(json.dumps({"config": wl.name, "n_gpus": world, "tokens_per_gpu": a.tokens, "buckets": B,
                      "compute_tflop_per_iter": 3 * sum(reps_f) * gemm_flops / 1e12,
                      "ms_compute": res["compute"], "ms_serial": res["serial"],
                      "ms_serial_buckets": res["serial_buckets"], "K": K, "cap": a.cap or wl.cap,
                      "ms_compute_with_carveout": {k: v for k, v in res.items() if k.startswith("compute_carveout")},
                      "ms_compute_on_partition": {k: v for k, v in res.items() if k.startswith("compute_green")},
                      "ms_overlap_by_max_ctas": over, "best_max_ctas": best, "ms_overlap": over[best],
                      "exposed_ms_serial": exposed_serial, "exposed_ms_overlap": exposed_overlap,
                      "hidden_frac": 1.0 - exposed_overlap / exposed_serial if exposed_serial > 0 else None,
                      "ms_ce": res.get("ce"),
                      "exposed_ms_ce": (res["ce"] - res["compute"]) if "ce" in res else None,
                      "ce_phases_ms_rank0": ce_phases if world > 1 else None}))
L.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
