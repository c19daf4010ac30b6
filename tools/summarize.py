"""Print a compact table from bench JSON lines (interleaved with {"run"/"tune": ...} markers)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        try:
            d = json.loads(line)
        except Exception:
            continue
        if "run" in d or "tune" in d:
            print(d.get("run") or d.get("tune"))
            continue
        if "roofline" not in d:
            print("  ", line[:200])
            continue
        r, p = d["roofline"], d["phases_ms"]
        ra, rb = r["pass_a"], r["pass_b"]
        print("  ms %.3f  %.1f Gp/s  A %.3f ms %.0f GB/s nvl %s  B %.3f ms %.0f GB/s nvl %s  roof %s %.3f" % (
            d["ms_per_step"], d["value"] / 1e9, p["pass_a"], ra["GBps"], ra.get("nvlink_frac"), p["pass_b"],
            rb["GBps"], rb.get("nvlink_frac"), r["bound"], r["frac"]))
