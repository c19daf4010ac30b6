#!/usr/bin/env python
"""Bench: sharded LAMB step (MegaScale arXiv 2402.15627 DP hot path) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt1.3b] [--comm fused|nccl]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle arm (bounded sample, host cores)

Metric (BASELINE.json): LAMB params updated/sec & step ms at 1/2/4/8 B200; % HBM roofline.
One step = one lamb_step (rows a1-a6 of SURVEY.md §8(a)) over the whole parameter table,
inputs resident in HBM (state >> L2, so no flush is needed).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "LAMB params updated/sec & step ms at 1/2/4/8 B200; % HBM roofline"
UNIT = "params/s"
FALLBACK_HBM_GBS = 6650.0
# NVLink roofline for the fused passes: B200_PROFILING.md prescribes "bytes that must cross
# NVLink / link bandwidth, the measured 770 GB/s per direction per GPU".  (Context: an LDG-based
# all-to-all on this pool reaches 633 GB/s pull / 700 GB/s push per GPU, tools/p2p_bench.cu,
# profiles/r01/p2p_all2all_D*.json; the TMA pass A already pulls ~670 GB/s.)
NVLINK_PEER_GBS = 770.0
NVLINK_PULL_GBS = NVLINK_PEER_GBS
NVLINK_PUSH_GBS = NVLINK_PEER_GBS


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt1.3b", choices=list(W.CONFIGS))
    ap.add_argument("--comm", default="fused", choices=["fused", "nccl"])
    ap.add_argument("--clip", type=float, default=0.0,
                    help="enable the NEXT #3 pre-step with this max grad norm (0 = off)")
    ap.add_argument("--graph", action="store_true", help="replay the step as one CUDA graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample time")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy r+w)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ oracle (CPU) timing
def oracle_sample(wl, seconds: float, max_steps: int | None = None, warmup: int = 0):
    """Time the CPU oracle's LAMB step on a bounded sample of the workload: the first
    transformer layer's tensors (or the first tensors up to ~50M params), repeated steps.
    Returns (params_per_s, ms_per_step, cores, sample description, steps)."""
    import numpy as np
    import oracle
    ids, n = [], 0
    for i, t in enumerate(wl.tensors):
        if t.name == "emb":
            continue
        ids.append(i)
        n += t.numel
        if n >= 60_000_000 or (t.name.endswith("fc2.b") and n >= 5_000_000):
            break
    wd = {i: oracle.gen_weights(wl.seed, i, wl.tensors[i].init, wl.tensors[i].numel) for i in ids}
    md = {i: np.zeros(wl.tensors[i].numel) for i in ids}
    vd = {i: np.zeros(wl.tensors[i].numel) for i in ids}
    gd = {i: oracle.gen_grads(wl.seed, 1, i, 1, wl.tensors[i].gexp, wl.tensors[i].numel) for i in ids}
    times = []
    t = 0
    while True:
        t += 1
        t0 = time.perf_counter()
        for i in ids:
            oracle.lamb_tensor_step(wd[i], md[i], vd[i], gd[i], wl.groups[wl.tensors[i].group], t)
        dt = time.perf_counter() - t0
        if t > warmup:
            times.append(dt)
        if max_steps is not None and len(times) >= max_steps:
            break
        if max_steps is None and sum(times) >= seconds and len(times) >= 2:
            break
    ms = 1e3 * statistics.mean(times)
    desc = (f"{wl.name}: tensors {ids[0]}..{ids[-1]} ({n / 1e6:.1f}M params, first layer), "
            f"{len(times)} LAMB steps in double, grads pre-generated")
    return n / (ms / 1e3), ms, oracle.num_threads(), desc, len(times)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = W.get(args.config)
    v, ms, cores, desc, k = oracle_sample(wl, 0, max_steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "sample": desc},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = nvml_handle(pynvml, device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ our arm
def nvml_handle(pynvml, device: int):
    """NVML handle of CUDA device `device` (matched by UUID: CUDA and NVML orders may differ)."""
    import torch
    try:
        return pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(device).uuid))
    except Exception:
        return pynvml.nvmlDeviceGetHandleByIndex(device)


def bind_numa_local(device: int):
    """Pin this rank to the CPUs NVML reports as local to its GPU, so the pinned host buffers of
    the e2e leg are first-touched on the GPU's NUMA node (one rank per GPU share the host)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = nvml_handle(pynvml, device)
        n = (os.cpu_count() + 63) // 64
        words = pynvml.nvmlDeviceGetCpuAffinity(h, n)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD

    from paper_2402_15627_b200 import lamb
    wl = W.get(args.config)
    spec = [(t.init, t.gexp) for t in wl.tensors]
    comm = lamb.LAMB_COMM_FUSED if args.comm == "fused" else lamb.LAMB_COMM_NCCL
    L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, world_size=world, rank=rank,
                  device=local, comm_mode=comm, bucket_cap=wl.cap, timing=not args.graph, pg=pg,
                  graph=args.graph)
    L.synth_init(spec, wl.seed)
    L.synth_grads(spec, wl.seed, rank + 1, 1)      # PER_RANK gradients, resident in HBM
    if args.clip > 0:
        L.set_grad_clip(args.clip)
    stream = torch.cuda.current_stream()
    K, Wm = args.steps, args.warmup

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for t in range(1, Wm + 1):
        L.step(t)
    barrier()
    if not args.graph:
        L.timing_begin(K)
    n0 = L.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        h0 = time.perf_counter()
        for t in range(Wm + 1, Wm + K + 1):
            L.step(t)
        host_us = (time.perf_counter() - h0) / K * 1e6   # host enqueue cost per step (async)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = L.launch_count() - n0
    ms_local = e0.elapsed_time(e1) / K
    if args.graph:   # no per-phase events inside a graph: attribute the step to the passes by bytes
        ph_mean = np.zeros(6)
        ph_mean[1] = ph_mean[4] = ms_local / 2
    else:
        ph = L.timing_read()                  # [K][6] ms per phase, events on the launch stream
        ph_mean = ph.mean(axis=0)
    ms = ms_local
    if world > 1:
        tt = torch.tensor([ms_local] + list(ph_mean), dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
        ph_mean = tt[1:].cpu().numpy()

    # ---------------- e2e: host buffers through lamb_step_host (H2D grads + D2H params in region)
    e2e = None
    if not args.no_e2e:
        numa_cpus = bind_numa_local(local) if world > 1 and os.environ.get("LAMB_BENCH_NUMA", "1") != "0" else None
        flat = L.plan.flat_size
        hg = torch.empty(flat, dtype=torch.bfloat16, pin_memory=True)
        hg.copy_(L.grad_buffer())
        hp = torch.empty(flat, dtype=torch.bfloat16, pin_memory=True)
        Ke = max(3, min(K, 20))
        L.step_host(hg, hp, Wm + K + 1)
        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for t in range(Wm + K + 2, Wm + K + 2 + Ke):
            L.step_host(hg, hp, t)
        e3.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e2.elapsed_time(e3) / Ke
        if world > 1:
            tt = torch.tensor([ms_e2e], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_e2e = float(tt[0])
        e2e = {"value": wl.n_params / (ms_e2e / 1e3), "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": 2 * flat * world, "d2h_bytes_per_step": 2 * flat * world,
               "steps": Ke, "api": "lamb_step_host (pinned host grads in, params out)",
               "numa_local_cpus": numa_cpus}

    if rank != 0:
        L.close()
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel (algorithmic bytes)
    hbm, hbm_src = peaks()
    owned = int(sum(s[3] for s in L.plan.segments.tolist()))   # tensor elements this rank owns
    D = world
    fused = D > 1 and comm == lamb.LAMB_COMM_FUSED
    n_flat = int(L.plan.flat_size)
    # local HBM bytes per launch: own state (w r, m rw, v rw = 20 B) + gradients: D = 1 reads its
    # bf16 grads (2 B); FUSED reads its whole flat grad buffer once across all D readers (2 B x
    # flat / owned per element); NCCL mode reads the fp32 reduced shard (4 B)
    grad_b = 2 * owned if D == 1 else (2 * n_flat if fused else 4 * owned)
    bytes_a = 20 * owned + grad_b
    bytes_b = 16 * owned + (2 * n_flat if fused else 2 * owned)   # m r, v r, w rw + params written
    nvl_in = 2 * owned * (D - 1) if fused else 0                  # NVLink in per GPU per pass
    t_a, t_b = float(ph_mean[1]), float(ph_mean[4])

    def pass_roof(name, nbytes, ms, nvl_peak):
        hbm_gbps = nbytes / (ms / 1e3) / 1e9
        out = {"kernel": name, "ms": ms, "bytes": nbytes, "GBps": hbm_gbps, "hbm_frac": hbm_gbps / hbm}
        if nvl_in:
            nvl_gbps = nvl_in / (ms / 1e3) / 1e9
            out.update({"nvlink_in_bytes": nvl_in, "nvlink_GBps": nvl_gbps, "nvlink_peak": nvl_peak,
                        "nvlink_frac": nvl_gbps / nvl_peak})
        # the binding resource: the one whose bytes need the longer time at its peak
        out["bound"] = "nvlink" if nvl_in and nvl_in / nvl_peak > nbytes / hbm else "hbm"
        return out

    if args.graph:
        # no per-kernel events inside a replayed graph: the whole step against its HBM bytes
        nvl_in = 0
        ra = rb = dom = pass_roof("step(graph)", bytes_a + bytes_b, ms, NVLINK_PULL_GBS)
    else:
        ra = pass_roof("pass_a", bytes_a, t_a, NVLINK_PULL_GBS)
        rb = pass_roof("pass_b", bytes_b, t_b, NVLINK_PUSH_GBS)
        dom = ra if t_a >= t_b else rb
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        d = json.load(open(tp)).get(f"{wl.name}/D{D}/{args.comm if D > 1 else 'fused'}/{dom['kernel']}")
        traffic = d["bytes"] if d else None
    if dom["bound"] == "nvlink":
        roof = {"bound": "nvlink", "kernel": dom["kernel"], "achieved": dom["nvlink_GBps"],
                "peak": dom["nvlink_peak"], "unit": "GB/s", "frac": dom["nvlink_frac"],
                "traffic": traffic,
                "peak_source": "B200_PROFILING.md measured peer copy, 770 GB/s per direction per GPU"}
    else:
        roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["GBps"], "peak": hbm,
                "unit": "GB/s", "frac": dom["hbm_frac"], "traffic": traffic, "peak_source": hbm_src}
    roof.update({"algorithmic_bytes_per_launch": dom["bytes"], "launch_ms": dom["ms"],
                 "pass_a": ra, "pass_b": rb,
                 "step_compulsory_frac": (owned * 28 / (ms / 1e3) / 1e9) / hbm})
    if D > 1:
        nvl = 2 * owned * (D - 1) * 2   # bytes in per GPU: peers' grads (RS) + peers' params (AG)
        roof["nvlink"] = {"bytes_in_per_gpu": nvl, "GBps_step": nvl / (ms / 1e3) / 1e9,
                          "peak_per_direction": NVLINK_PEER_GBS,
                          "frac_step": nvl / (ms / 1e3) / 1e9 / NVLINK_PEER_GBS}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, cms, cores, desc, k = oracle_sample(wl, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
               "ms_per_sample_step": cms}

    line = {"metric": METRIC, "value": wl.n_params / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Philox4x32-10 grads/weights, DESIGN.md §4)",
            "config": {"workload": wl.name, "n_params": wl.n_params, "n_tensors": len(wl.tensors),
                       "flat_size": L.plan.flat_size, "world_size": world,
                       "comm": args.comm if world > 1 else "none", "bucket_cap": wl.cap,
                       "prestep_clip": args.clip if args.clip > 0 else None,
                       "cuda_graph": bool(args.graph),
                       "l2": "inputs larger than L2 (fp32 state of the shard >> 126 MB)",
                       "io_dtype": "bf16 grads in / bf16 params out, fp32 master and moments",
                       "parallelism": f"zero2-dp{world}"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "host_enqueue_us_per_step": host_us,
            "clocks": clk.summary(),
            "phases_ms": {n: float(x) for n, x in zip(lamb.PHASES, ph_mean)}}
    print(json.dumps(line), flush=True)
    L.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
