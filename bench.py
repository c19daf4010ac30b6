#!/usr/bin/env python
"""Bench: sharded LAMB step (MegaScale arXiv 2402.15627 DP hot path) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt1.3b] [--comm fused|nccl]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle arm (bounded sample, host cores)

`--gpus N > 1` without torchrun re-launches itself as N ranks through torch.distributed.run
(127.0.0.1); under torchrun it runs as the rank the environment names.

Metric (BASELINE.json): LAMB params updated/sec & step ms at 1/2/4/8 B200; % HBM roofline.
One step = one lamb_step (rows a1-a6 of SURVEY.md §8(a)) over the whole parameter table,
inputs resident in HBM (state >> L2, so no flush is needed).  Prints ONE JSON line on rank 0.
The main value is the `--config` workload (default: BASELINE configs[1], GPT 1.3B layout);
`north_star_curve` adds the north star's scaling-curve layout (175B slice, 3 layers) timed the
same way after the main handle is freed (`--no-curve` skips it).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
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
# Context for the NVLink fractions: what an all-to-all actually reaches on this fabric (no
# compute, per GPU, user data) — TMA bulk pulls 658-669 GB/s at D = 4 (tools/p2p_bench.cu mode 1,
# profiles/r02/p2p_tma_pull_D4_D2.jsonl), STG pushes 695-700 GB/s (profiles/r01/p2p_all2all_D4.json)
ALLTOALL_PULL_GBS = 669.0
ALLTOALL_PUSH_GBS = 700.0
CURVE_CONFIG = "175b_slice_3l"     # north_star: "1->8 GPU step-time scaling curve on the 175B-slice layout"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt1.3b", choices=list(W.CONFIGS))
    ap.add_argument("--comm", default="fused", choices=["fused", "nccl", "nvls"])
    ap.add_argument("--clip", type=float, default=0.0,
                    help="enable the NEXT #3 pre-step with this max grad norm (0 = off)")
    ap.add_argument("--graph", action="store_true", help="replay the step as one CUDA graph")
    ap.add_argument("--pg", default="nccl", choices=["nccl", "gloo"],
                    help="process group of the harness; gloo also bootstraps the library without NCCL "
                         "(lamb_create_with_allgather) — e.g. for an ncu capture of rank 0")
    ap.add_argument("--max-ctas", type=int, default=0, help="cap the persistent grids (lamb_set_max_ctas; 0 = full)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-curve", action="store_true", help="skip the 175B-slice-3L curve point")
    ap.add_argument("--curve-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample time")
    ap.add_argument("--cpu-probe", action="store_true", help=argparse.SUPPRESS)  # internal: 1-core leg
    return ap.parse_args(argv)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy r+w)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ oracle (CPU) timing
def sample_ids(wl):
    """The bounded oracle sample: the first transformer layer's tensors (embedding skipped), or
    the first tensors up to ~60M params."""
    ids, n = [], 0
    for i, t in enumerate(wl.tensors):
        if t.name == "emb":
            continue
        ids.append(i)
        n += t.numel
        if n >= 60_000_000 or (t.name.endswith("fc2.b") and n >= 5_000_000):
            break
    return ids, n


def oracle_time(wl, ids, seconds: float, max_steps: int | None = None, warmup: int = 0):
    """Time the CPU oracle's LAMB step (as it stands) over tensors `ids` of `wl`, repeated steps,
    grads pre-generated.  Returns (mean ms per step, steps timed)."""
    import numpy as np
    import oracle
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
    return 1e3 * statistics.mean(times), len(times)


def oracle_sample(wl, seconds: float, max_steps: int | None = None, warmup: int = 0):
    """Oracle params/s on the bounded sample.  Returns (params_per_s, ms_per_step, cores,
    sample description, steps)."""
    import oracle
    ids, n = sample_ids(wl)
    ms, k = oracle_time(wl, ids, seconds, max_steps, warmup)
    desc = (f"{wl.name}: tensors {ids[0]}..{ids[-1]} ({n / 1e6:.1f}M params, first layer), "
            f"{k} LAMB steps in double, grads pre-generated")
    return n / (ms / 1e3), ms, oracle.num_threads(), desc, k


def cpu_model() -> str | None:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_probe(wl, seconds: float) -> dict:
    """One oracle leg with whatever OpenMP thread count the environment gives: the workload's
    sample (params/s) and the full toy step (ms).  Used on all cores in-process and on 1 core in a
    subprocess (OMP_NUM_THREADS=1), so the oracle itself is never modified for the timing."""
    import oracle
    v, ms, cores, desc, k = oracle_sample(wl, seconds)
    toy = W.toy()
    toy_ms, toy_k = oracle_time(toy, list(range(len(toy.tensors))), min(1.0, seconds / 4), warmup=2)
    return {"value": v, "ms_per_sample_step": ms, "cores": cores, "sample": desc, "steps": k,
            "toy_full_step_ms": toy_ms, "toy_steps": toy_k, "threads": oracle.num_threads()}


def cpu_leg(wl, seconds: float, threads: int) -> dict:
    """Run cpu_probe in a fresh process with OMP_NUM_THREADS=threads (torchrun sets 1 for its
    ranks, and the e2e leg may have pinned this rank to a NUMA node's CPUs)."""
    try:
        env = dict(os.environ, OMP_NUM_THREADS=str(threads))
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-probe", "--config", wl.name,
                            "--cpu-seconds", str(seconds)], capture_output=True, text=True,
                           timeout=900, env=env, cwd=ROOT)
        if r.returncode == 0:
            return json.loads(r.stdout.strip().splitlines()[-1])
        return {"error": r.stderr[-300:]}
    except Exception as e:  # pragma: no cover
        return {"error": repr(e)}


def cpu_baseline(wl, seconds: float) -> dict:
    """SURVEY §8(d) 'Oracle timing': the oracle on all host cores and on 1 core; the sample's
    params/s, the full toy step, and the workload's full step extrapolated from the sample
    (labelled: the per-element work of LAMB is uniform, the norms are per tensor)."""
    allc = cpu_leg(wl, seconds, os.cpu_count() or 1)
    if "value" not in allc:
        return {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "error": allc.get("error")}
    one = cpu_leg(wl, max(2.0, seconds / 3), 1)
    out = {"value": allc["value"], "unit": UNIT, "cores": allc["cores"], "kind": "oracle",
           "sample": allc["sample"], "ms_per_sample_step": allc["ms_per_sample_step"],
           "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
           "toy_full_step_ms": allc["toy_full_step_ms"],
           "full_step_ms": 1e3 * wl.n_params / allc["value"], "extrapolated": True,
           "extrapolation": f"{wl.name} full step = n_params / sample params/s (sample above)"}
    if one and "value" in one:
        out.update({"value_1core": one["value"], "ms_per_sample_step_1core": one["ms_per_sample_step"],
                    "cores_1core": one["cores"], "toy_full_step_ms_1core": one["toy_full_step_ms"],
                    "full_step_ms_1core": 1e3 * wl.n_params / one["value"]})
    else:
        out["one_core_error"] = one
    return out


def run_config(args, wl, world: int, flat_size: int) -> dict:
    """The `config` object of the JSON line — identical for our arm and the reference arm (the
    reference times a bounded sample of this same workload; the sample is described in its
    cpu_baseline)."""
    return {"workload": wl.name, "n_params": wl.n_params, "n_tensors": len(wl.tensors),
            "flat_size": flat_size, "world_size": world,
            "comm": args.comm if world > 1 else "none", "bucket_cap": wl.cap,
            "prestep_clip": args.clip if args.clip > 0 else None,
            "cuda_graph": bool(args.graph), "max_ctas": args.max_ctas or None,
            "l2": "inputs larger than L2 (fp32 state of the shard >> 126 MB)",
            "io_dtype": "bf16 grads in / bf16 params out, fp32 master and moments",
            "parallelism": f"zero2-dp{world}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    wl = W.get(args.config)
    v, ms, cores, desc, k = oracle_sample(wl, 0, max_steps=args.steps, warmup=args.warmup)
    flat = oracle.plan([t.numel for t in wl.tensors], args.gpus, wl.cap).flat_size   # oracle planner
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox4x32-10 grads/weights, DESIGN.md §4); the CPU oracle (double) on a "
                    "bounded sample of the workload: " + desc,
            "config": run_config(args, wl, args.gpus, flat),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             "cpu_model": cpu_model()},
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


class NvlinkCounters:
    """NVML NVLink data counters of one GPU, summed over its links: bytes transmitted and
    received.  Tries the per-link byte counters (NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES) and
    falls back to the throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB).
    `read()` returns (tx_bytes, rx_bytes) or None when neither is available."""
    N_LINKS = 18

    def __init__(self, device: int):
        self.ok, self.field, self.scale = False, None, 1
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nvml_handle(nv, device)
            cands = []
            if hasattr(nv, "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES"):
                cands.append(("COUNT_XMIT/RCV_BYTES", nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                              nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1))
            if hasattr(nv, "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX"):
                cands.append(("THROUGHPUT_DATA_TX/RX (KiB)", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                              nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024))
            for name, ftx, frx, scale in cands:
                self.ftx, self.frx, self.scale, self.field = ftx, frx, scale, name
                if self._read_raw() is not None:
                    self.ok = True
                    break
        except Exception:
            self.ok = False

    def _read_raw(self):
        nv = self.nv
        req = [(self.ftx, l) for l in range(self.N_LINKS)] + [(self.frx, l) for l in range(self.N_LINKS)]
        vals = nv.nvmlDeviceGetFieldValues(self.h, req)
        tx = rx = 0
        good = 0
        for k, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            x = int(v.value.ullVal)
            good += 1
            if k < self.N_LINKS:
                tx += x
            else:
                rx += x
        return (tx * self.scale, rx * self.scale) if good else None

    def read(self):
        if not self.ok:
            return None
        try:
            return self._read_raw()
        except Exception:
            return None


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


def self_launch(args) -> int:
    """`--gpus N > 1` outside torchrun: run this same command as N ranks, one per GPU, through
    torch.distributed.run on 127.0.0.1 (the driver's launch form).  Rank 0's JSON line goes
    straight to stdout."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Run:
    """Timing of one workload on this rank: create the handle, synth state/grads in HBM, W
    warm-up steps, K timed steps bracketed by barrier + synchronize (CUDA events on the launch
    stream, per-phase events from the library, NVML clocks and NVLink counters around the
    region), max over ranks."""

    def __init__(self, wl, args, world, rank, local, pg):
        import torch
        from paper_2402_15627_b200 import lamb
        self.wl, self.world, self.rank, self.local, self.pg = wl, world, rank, local, pg
        self.lamb = lamb
        self.comm = {"fused": lamb.LAMB_COMM_FUSED, "nccl": lamb.LAMB_COMM_NCCL, "nvls": lamb.LAMB_COMM_NVLS}[args.comm]
        spec = [(t.init, t.gexp) for t in wl.tensors]
        self.L = lamb.Lamb([(t.numel, t.group) for t in wl.tensors], wl.groups, world_size=world, rank=rank,
                           device=local, comm_mode=self.comm, bucket_cap=wl.cap, timing=not args.graph, pg=pg,
                           graph=args.graph, bootstrap="host" if args.pg == "gloo" and world > 1 else "nccl")
        if args.max_ctas > 0:
            self.L.set_max_ctas(args.max_ctas)
        self.L.synth_init(spec, wl.seed)
        self.L.synth_grads(spec, wl.seed, rank + 1, 1)      # PER_RANK gradients, resident in HBM
        if args.clip > 0:
            self.L.set_grad_clip(args.clip)
        self.stream = torch.cuda.current_stream()
        self.graph = args.graph

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, vals):
        import numpy as np
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return np.asarray(vals, dtype=np.float64)
        tt = torch.tensor(list(vals), dtype=torch.float64, device=_pg_device())
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return tt.cpu().numpy()

    def time(self, K: int, Wm: int, t0: int = 1):
        import numpy as np
        import torch
        L = self.L
        for t in range(t0, t0 + Wm):
            L.step(t)
        self.barrier()
        if not self.graph:
            L.timing_begin(K)
        n0 = L.launch_count()
        nvc = NvlinkCounters(self.local) if self.world > 1 else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(self.local) as clk:
            self.barrier()
            c0 = nvc.read() if nvc else None
            e0.record(self.stream)
            h0 = time.perf_counter()
            for t in range(t0 + Wm, t0 + Wm + K):
                L.step(t)
            host_us = (time.perf_counter() - h0) / K * 1e6   # host enqueue cost per step (async)
            e1.record(self.stream)
            torch.cuda.synchronize()
            c1 = nvc.read() if nvc else None
        self.barrier()
        self.t_next = t0 + Wm + K
        self.launches = L.launch_count() - n0
        ms_local = e0.elapsed_time(e1) / K
        if self.graph:   # no per-phase events inside a graph: attribute the step to the passes by bytes
            ph = np.zeros(6)
            ph[1] = ph[4] = ms_local / 2
        else:
            ph = L.timing_read().mean(axis=0)       # [K][6] ms per phase, events on the launch stream
        m = self.max_over_ranks([ms_local] + list(ph))
        self.ms, self.ph = float(m[0]), m[1:]
        self.host_us, self.clocks = host_us, clk.summary()
        self.nvlink_meas = None
        if nvc is not None:
            if c0 is not None and c1 is not None:
                tx, rx = (c1[0] - c0[0]) / K, (c1[1] - c0[1]) / K
                mm = self.max_over_ranks([tx, rx, -tx, -rx])
                self.nvlink_meas = {"field": nvc.field, "tx_bytes_per_step_rank0": tx,
                                    "rx_bytes_per_step_rank0": rx,
                                    "tx_bytes_per_step_max": float(mm[0]), "rx_bytes_per_step_max": float(mm[1]),
                                    "tx_bytes_per_step_min": float(-mm[2]), "rx_bytes_per_step_min": float(-mm[3])}
            else:
                self.max_over_ranks([0, 0, 0, 0])
                self.nvlink_meas = {"field": None, "note": "NVML NVLink byte counters unavailable"}

    def roofline(self, args):
        """Algorithmic-byte roofline of the dominant pass."""
        L, D = self.L, self.world
        hbm, hbm_src = peaks()
        owned = int(sum(s[3] for s in L.plan.segments.tolist()))   # tensor elements this rank owns
        # FUSED and NVLS touch the same local HBM bytes: own state, plus this rank's whole flat
        # grad buffer read once (by the D readers / by the switch) and its whole param buffer
        # written once (by the D writers / by the switch)
        fused = D > 1 and self.comm in (self.lamb.LAMB_COMM_FUSED, self.lamb.LAMB_COMM_NVLS)
        n_flat = int(L.plan.flat_size)
        # local HBM bytes per launch: own state (w r, m rw, v rw = 20 B) + gradients: D = 1 reads its
        # bf16 grads (2 B); FUSED reads its whole flat grad buffer once across all D readers (2 B x
        # flat / owned per element); NCCL mode reads the fp32 reduced shard (4 B)
        grad_b = 2 * owned if D == 1 else (2 * n_flat if fused else 4 * owned)
        bytes_a = 20 * owned + grad_b
        bytes_b = 16 * owned + (2 * n_flat if fused else 2 * owned)   # m r, v r, w rw + params written
        # NVLink bytes per GPU per pass in the busier direction: FUSED pulls (A) / pushes (B) the
        # D-1 peers' slices, 2(D-1) B per owned element each way; NVLS (switch-side reduce /
        # multicast store) sends this rank's whole grad buffer to the switch (A, out) and receives
        # every rank's params (B, in): 2 B per flat element
        nvls = D > 1 and self.comm == self.lamb.LAMB_COMM_NVLS
        nvl_in = (2 * n_flat if nvls else 2 * owned * (D - 1)) if fused else 0
        t_a, t_b = float(self.ph[1]), float(self.ph[4])
        ms = self.ms

        def pass_roof(name, nbytes, t, nvl_peak, nvl):
            hbm_gbps = nbytes / (t / 1e3) / 1e9
            out = {"kernel": name, "ms": t, "bytes": nbytes, "GBps": hbm_gbps, "hbm_frac": hbm_gbps / hbm}
            if nvl:
                nvl_gbps = nvl / (t / 1e3) / 1e9
                out.update({"nvlink_in_bytes": nvl, "nvlink_GBps": nvl_gbps, "nvlink_peak": nvl_peak,
                            "nvlink_frac": nvl_gbps / nvl_peak})
            # the binding resource: the one whose bytes need the longer time at its peak
            out["bound"] = "nvlink" if nvl and nvl / nvl_peak > nbytes / hbm else "hbm"
            return out

        if self.graph:
            # no per-kernel events inside a replayed graph: the whole step against its HBM bytes
            ra = rb = dom = pass_roof("step(graph)", bytes_a + bytes_b, ms, NVLINK_PULL_GBS, 0)
        else:
            ra = pass_roof("pass_a", bytes_a, t_a, NVLINK_PULL_GBS, nvl_in)
            rb = pass_roof("pass_b", bytes_b, t_b, NVLINK_PUSH_GBS, nvl_in)
            dom = ra if t_a >= t_b else rb
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            d = json.load(open(tp)).get(f"{self.wl.name}/D{D}/{args.comm if D > 1 else 'fused'}/{dom['kernel']}")
            traffic = d["bytes"] if d else None
        if dom["bound"] == "nvlink":
            roof = {"bound": "nvlink", "kernel": dom["kernel"], "achieved": dom["nvlink_GBps"],
                    "peak": dom["nvlink_peak"], "unit": "GB/s", "frac": dom["nvlink_frac"],
                    "traffic": traffic,
                    "peak_source": "B200_PROFILING.md measured peer copy, 770 GB/s per direction per GPU",
                    "alltoall_ceiling": {"GBps": ALLTOALL_PULL_GBS if dom["kernel"] == "pass_a" else ALLTOALL_PUSH_GBS,
                                         "frac": dom["nvlink_GBps"] / (ALLTOALL_PULL_GBS if dom["kernel"] == "pass_a"
                                                                      else ALLTOALL_PUSH_GBS),
                                         "source": "measured all-to-all (no compute) on this pool: TMA pulls / "
                                                   "STG pushes, DESIGN.md §11b"}}
        else:
            roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["GBps"], "peak": hbm,
                    "unit": "GB/s", "frac": dom["hbm_frac"], "traffic": traffic, "peak_source": hbm_src}
        roof.update({"algorithmic_bytes_per_launch": dom["bytes"], "launch_ms": dom["ms"],
                     "pass_a": ra, "pass_b": rb,
                     "step_compulsory_frac": (owned * 28 / (ms / 1e3) / 1e9) / hbm})
        if D > 1:
            # algorithmic NVLink bytes per GPU per step, each direction: peers' grads pulled by this
            # rank (RS) + peers' params stored into this rank (AG) = 4 B x owned x (D-1) in; the
            # same amount out (this rank's grads pulled by peers + its params stored into peers)
            nvl = (2 * n_flat * 2 if nvls else 2 * owned * (D - 1) * 2) if fused else None
            roof["nvlink"] = {"bytes_in_per_gpu": nvl, "GBps_step": nvl / (ms / 1e3) / 1e9 if nvl else None,
                              "peak_per_direction": NVLINK_PEER_GBS,
                              "frac_step": nvl / (ms / 1e3) / 1e9 / NVLINK_PEER_GBS if nvl else None,
                              "traffic": self.nvlink_meas}
            if nvl and self.nvlink_meas and self.nvlink_meas.get("rx_bytes_per_step_rank0") is not None:
                roof["nvlink"]["measured_over_algorithmic_rx"] = self.nvlink_meas["rx_bytes_per_step_rank0"] / nvl
                roof["nvlink"]["measured_over_algorithmic_tx"] = self.nvlink_meas["tx_bytes_per_step_rank0"] / nvl
            # per-kernel NVLink bytes measured by ncu (nvlrx/nvltx; one process driving the D GPUs,
            # tools/nvlink_bytes_1proc.py -> profiles/ncu_nvlink.json): user data and wire bytes of
            # the busier direction of each pass against the algorithmic bytes
            tp = os.path.join(ROOT, "profiles", "ncu_nvlink.json")
            meas = json.load(open(tp)) if os.path.exists(tp) else {}
            per_pass = {}
            for name, key, d_user, d_wire in (("pass_a", "pass_a", "nvlink_rx_user_bytes", "nvlink_rx_bytes"),
                                              ("pass_b", "pass_b", "nvlink_tx_user_bytes", "nvlink_tx_bytes")):
                e = meas.get(f"{self.wl.name}/D{D}/{args.comm}/{key}")
                if e and e.get(d_user) and nvl_in:
                    per_pass[name] = {"algorithmic_bytes": nvl_in, "ncu_user_bytes": e[d_user],
                                      "ncu_wire_bytes": e[d_wire], "user_over_algorithmic": e[d_user] / nvl_in,
                                      "wire_over_algorithmic": e[d_wire] / nvl_in,
                                      "direction": "rx (pulls)" if name == "pass_a" else "tx (pushes)",
                                      "source": "profiles/ncu_nvlink.json (" + e["source"] + ")"}
            roof["nvlink"]["ncu_traffic"] = per_pass or None
        return roof

    def close(self):
        self.L.close()


def _pg_device():
    """Device of the tensors the harness's collectives use (gloo: host)."""
    import torch.distributed as dist
    return "cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else "cuda"


def ranks_seen(world: int) -> int:
    """Distinct GPUs (device UUIDs) across the ranks of this run."""
    import torch
    import torch.distributed as dist
    u = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
    if world == 1:
        return 1
    out = [None] * world
    dist.all_gather_object(out, u)
    return len(set(out))


def main():
    args = parse()
    if args.cpu_probe:
        try:   # every host CPU (a parent may have been pinned to one NUMA node)
            os.sched_setaffinity(0, set(range(os.cpu_count() or 1)))
        except OSError:
            pass
        print(json.dumps(cpu_probe(W.get(args.config), args.cpu_seconds)), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    # stdout carries exactly ONE line (the JSON result): native libraries that print on fd 1
    # (e.g. NCCL's version banner on rank 0) are sent to stderr instead
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
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
        if args.pg == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    n_seen = ranks_seen(world)

    wl = W.get(args.config)
    K, Wm = args.steps, args.warmup
    R = Run(wl, args, world, rank, local, pg)
    R.time(K, Wm)
    L = R.L

    # ---------------- e2e: host buffers through lamb_step_host (H2D grads + D2H params in region)
    e2e = None
    if not args.no_e2e:
        numa_cpus = bind_numa_local(local) if world > 1 and os.environ.get("LAMB_BENCH_NUMA", "1") != "0" else None
        flat = L.plan.flat_size
        hg = torch.empty(flat, dtype=torch.bfloat16, pin_memory=True)
        hg.copy_(L.grad_buffer())
        hp = torch.empty(flat, dtype=torch.bfloat16, pin_memory=True)
        Ke = max(3, min(K, 20))
        t = R.t_next
        L.step_host(hg, hp, t)
        R.barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(R.stream)
        for t in range(t + 1, t + 1 + Ke):
            L.step_host(hg, hp, t)
        e3.record(R.stream)
        torch.cuda.synchronize()
        ms_e2e = float(R.max_over_ranks([e2.elapsed_time(e3) / Ke])[0])
        e2e = {"value": wl.n_params / (ms_e2e / 1e3), "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": 2 * flat * world, "d2h_bytes_per_step": 2 * flat * world,
               "steps": Ke, "api": "lamb_step_host (pinned host grads in, params out)",
               "numa_local_cpus": numa_cpus}
        del hg, hp

    roof = R.roofline(args) if rank == 0 else None
    main_line = {"ms": R.ms, "ph": R.ph, "launches": R.launches, "host_us": R.host_us, "clocks": R.clocks,
                 "flat": L.plan.flat_size}
    R.close()
    del R, L
    torch.cuda.empty_cache()

    # ---------------- the north star's scaling-curve layout, timed the same way
    curve = None
    if not args.no_curve and args.config != CURVE_CONFIG and not args.graph:
        wc = W.get(CURVE_CONFIG)
        free, total = torch.cuda.mem_get_info()
        need = 4 * wc.n_params + 12 * wc.n_params // world + (1 << 30)
        ok = torch.tensor([1.0 if free >= need else 0.0], device=_pg_device())
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if float(ok[0]) > 0:
            Rc = Run(wc, args, world, rank, local, pg)
            Rc.time(max(3, args.curve_steps), max(3, min(Wm, 5)))
            rc = Rc.roofline(args)
            curve = {"workload": wc.name, "n_params": wc.n_params, "n_tensors": len(wc.tensors),
                     "value": wc.n_params / (Rc.ms / 1e3), "unit": UNIT, "ms_per_step": Rc.ms,
                     "steps": max(3, args.curve_steps), "phases_ms": {n: float(x) for n, x in zip(Rc.lamb.PHASES, Rc.ph)},
                     "roofline": {k: rc[k] for k in ("bound", "kernel", "achieved", "peak", "unit", "frac")},
                     "nvlink": rc.get("nvlink"), "clocks": Rc.clocks}
            Rc.close()
            del Rc
            torch.cuda.empty_cache()
        else:
            curve = {"workload": wc.name, "skipped": f"needs {need / 1e9:.1f} GB free per GPU, "
                                                     f"rank {rank} has {free / 1e9:.1f}"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_seconds)   # rank 0, after every timed region

    ms = main_line["ms"]
    from paper_2402_15627_b200 import lamb
    line = {"metric": METRIC, "value": wl.n_params / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Philox4x32-10 grads/weights, DESIGN.md §4)",
            "config": run_config(args, wl, world, main_line["flat"]),
            "ranks_seen": n_seen,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": main_line["launches"],
            "host_enqueue_us_per_step": main_line["host_us"],
            "clocks": main_line["clocks"],
            "phases_ms": {n: float(x) for n, x in zip(lamb.PHASES, main_line["ph"])},
            "north_star_curve": curve}
    print(json.dumps(line), file=out, flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
