"""Per-kernel NVLink bytes of the D-rank passes, for ncu: ONE process drives D handles on D GPUs
(one thread per rank, the C-ABI bootstrap through an in-process all-gather —
lamb_create_with_allgather), each rank takes ONE lamb_step.  Under ncu every kernel launch of the
process is serialised, so the cross-GPU barriers cannot meet: they are given a 200 ms bound
(LAMB_BARRIER_TIMEOUT_MS), time out, and the passes then run one at a time with their real
memory traffic (pass A pulls the peers' gradient slices / the switch reduces them, pass B stores
into every rank's param buffer) — the values are not checked, only the bytes are counted:

    LAMB_BARRIER_TIMEOUT_MS=200 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,\
        dram__bytes_write.sum,gpu__time_duration.sum -k regex:pass_ --csv --log-file out.csv \
        python tools/nvlink_bytes_1proc.py <D> <fused|nvls> [config]

(Multi-process ranks with rank 0 under ncu never got past their socket bootstrap on the gpurun
boxes, r02; NVML's NVLink byte counters answer NOT_SUPPORTED there.)  Tool, not product.
"""
import ctypes
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("LAMB_BARRIER_TIMEOUT_MS", "200")

import workloads as W  # noqa: E402
from paper_2402_15627_b200 import lamb as Lb  # noqa: E402


def main():
    D = int(sys.argv[1])
    mode = {"fused": Lb.LAMB_COMM_FUSED, "nvls": Lb.LAMB_COMM_NVLS}[sys.argv[2]]
    wl = W.get(sys.argv[3] if len(sys.argv) > 3 else "gpt1.3b")
    tensors = Lb._tensor_array([t.numel for t in wl.tensors], [t.group for t in wl.tensors])
    groups = (Lb.lamb_group * len(wl.groups))()
    for k, g in enumerate(wl.groups):
        groups[k].lr, groups[k].beta1, groups[k].beta2 = g.lr, g.beta1, g.beta2
        groups[k].eps, groups[k].weight_decay, groups[k].adapt, groups[k].bias_correction = \
            g.eps, g.weight_decay, g.adapt, g.bias_correction
    spec = (Lb.lamb_synth_tensor * len(wl.tensors))(*[Lb.lamb_synth_tensor(t.init, t.gexp) for t in wl.tensors])
    slots = [b""] * D
    bar = threading.Barrier(D)

    def make_ag(rank):
        def fn(send, recv, nbytes, _user):
            slots[rank] = ctypes.string_at(send, nbytes)
            bar.wait()
            for j in range(D):
                ctypes.memmove(recv + j * nbytes, slots[j], nbytes)
            bar.wait()
            return 0
        return Lb._ALLGATHER_FN(fn)

    handles = [None] * D
    errors = []

    def rank_main(r):
        try:
            import torch
            torch.cuda.set_device(r)
            cfg = Lb.lamb_config(D, r, r, mode, wl.cap, 0.0, 0)
            h = ctypes.c_void_p()
            ag = make_ag(r)
            st = Lb.lamb_create_with_allgather(tensors, len(wl.tensors), groups, len(wl.groups), ctypes.byref(cfg),
                                               ctypes.cast(ag, ctypes.c_void_p), None, ctypes.byref(h))
            if st != 0:
                raise RuntimeError(f"rank {r}: create failed: {Lb.lamb_last_error(None)}")
            handles[r] = h
            Lb.check(Lb.lamb_synth_init(h, spec, wl.seed, None), h)
            Lb.check(Lb.lamb_synth_grads(h, spec, wl.seed, r + 1, 1, None), h)
            torch.cuda.synchronize()
            bar.wait()
            Lb.lamb_step(h, None, 1, None)   # barriers time out under ncu (err flag); passes still run
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))
            bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(D)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for h in handles:
        if h is not None:
            Lb.lamb_destroy(h)
    print({"D": D, "mode": sys.argv[2], "workload": wl.name, "errors": errors}, flush=True)


if __name__ == "__main__":
    main()
