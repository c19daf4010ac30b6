"""Probe which NVML NVLink byte counters move, and by how much, for a known peer copy.

    python tools/nvlink_counter_probe.py      (needs >= 2 GPUs)

Reads every candidate NVML field (per device; per-link fields with scopeId = link) before and
after copying a known number of bytes from cuda:0 to cuda:1 (torch peer copy, copy engine) and
with an SM-driven peer store kernel-free path (torch .copy_ inside a kernel is CE) and prints
the deltas.  Output: one JSON line per experiment.
"""
import json
import os
import time

import pynvml as nv
import torch

nv.nvmlInit()
FIELDS = {n: getattr(nv, n) for n in dir(nv)
          if n.startswith("NVML_FI_DEV_NVLINK_") and any(k in n for k in ("THROUGHPUT", "XMIT_BYTES", "RCV_BYTES"))}


def handle(d):
    try:
        return nv.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(d).uuid))
    except Exception:
        return nv.nvmlDeviceGetHandleByIndex(d)


def read(h, nlinks=18, raw=None):
    out = {}
    for name, fid in FIELDS.items():
        for scope in [None] + list(range(nlinks)):
            try:
                if scope is None:
                    v = nv.nvmlDeviceGetFieldValues(h, [fid])[0]
                else:
                    v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                if raw is not None:
                    raw[f"{name}[{'dev' if scope is None else scope}]"] = (int(v.nvmlReturn), int(v.valueType))
                if v.nvmlReturn != 0:
                    continue
                val = v.value.ullVal if v.valueType in (3, 4) else v.value.uiVal
                out[f"{name}[{'dev' if scope is None else scope}]"] = int(val)
            except Exception as e:
                if raw is not None:
                    raw[f"{name}[{'dev' if scope is None else scope}]"] = repr(e)
    return out


def delta(a, b):
    return {k: b[k] - a[k] for k in b if k in a and b[k] != a[k]}


def main():
    n = torch.cuda.device_count()
    h = [handle(d) for d in range(n)]
    print(json.dumps({"ngpu": n, "fields": FIELDS, "cpu_count": os.cpu_count()}), flush=True)
    raw = {}
    vals = read(h[0], raw=raw)
    print(json.dumps({"raw_returns_gpu0": raw, "values_gpu0": vals}), flush=True)
    for fn in ("nvmlDeviceGetNvLinkState", "nvmlDeviceGetNvLinkVersion"):
        try:
            print(json.dumps({fn: [getattr(nv, fn)(h[0], l) for l in range(18)]}), flush=True)
        except Exception as e:
            print(json.dumps({fn: repr(e)}), flush=True)
    try:
        print(json.dumps({"util_counter_l0": list(nv.nvmlDeviceGetNvLinkUtilizationCounter(h[0], 0, 0))}), flush=True)
    except Exception as e:
        print(json.dumps({"util_counter_l0": repr(e)}), flush=True)
    nbytes = 1 << 30
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    dst.copy_(src)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for rep in range(2):
        time.sleep(1.0)
        a = [read(x) for x in h[:2]]
        for _ in range(4):
            dst.copy_(src)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        time.sleep(1.0)
        b = [read(x) for x in h[:2]]
        print(json.dumps({"experiment": f"4 x 1 GiB peer copy gpu0 -> gpu1 (rep {rep})", "bytes": 4 * nbytes,
                          "gpu0": delta(a[0], b[0]), "gpu1": delta(a[1], b[1])}), flush=True)
    time.sleep(1.0)
    a = [read(x) for x in h[:2]]
    time.sleep(1.0)
    b = [read(x) for x in h[:2]]
    print(json.dumps({"experiment": "idle 1 s", "gpu0": delta(a[0], b[0]), "gpu1": delta(a[1], b[1])}), flush=True)


if __name__ == "__main__":
    main()
