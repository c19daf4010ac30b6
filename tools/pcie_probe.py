"""Host-link ceiling for the e2e leg (lamb_step_host): pinned H2D alone, D2H alone, both at once,
and the same split over k streams per direction (more copy engines).  CUDA events, best of 5.

    python tools/pcie_probe.py [--gib 2.5]   -> one JSON line per variant
"""
import argparse
import json

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=2.5)
a = ap.parse_args()
n = int(a.gib * (1 << 30))
hin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hout = torch.empty(n, dtype=torch.uint8, pin_memory=True)
din = torch.empty(n, dtype=torch.uint8, device="cuda")
dout = torch.empty(n, dtype=torch.uint8, device="cuda")
hin.fill_(1)
dout.fill_(2)
streams = [torch.cuda.Stream() for _ in range(8)]


def run(h2d, d2h, k):
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record(cur)
        ss = []
        for i in range(k):
            lo, hi = n * i // k, n * (i + 1) // k
            if h2d:
                s = streams[i]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    din[lo:hi].copy_(hin[lo:hi], non_blocking=True)
                ss.append(s)
            if d2h:
                s = streams[4 + i]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    hout[lo:hi].copy_(dout[lo:hi], non_blocking=True)
                ss.append(s)
        for s in ss:
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    moved = n * (int(h2d) + int(d2h))
    print(json.dumps({"h2d": h2d, "d2h": d2h, "streams_per_dir": k, "bytes_per_dir": n, "ms": round(best, 3),
                      "GBps_total": round(moved / best / 1e6, 1),
                      "GBps_per_dir": round(n / best / 1e6, 1)}), flush=True)


for k in (1, 2, 4):
    run(True, False, k)
    run(False, True, k)
    run(True, True, k)
