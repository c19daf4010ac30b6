"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv>            -> per-kernel launch table
    python tools/ncu_summary.py full <report.ncu-rep> [algo.json]  -> key metrics per kernel
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("launch__grid_size", "grid"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    order = []
    for r in rows[1:]:
        n = r[ki].split("(")[0]
        if n not in tot:
            order.append(n)
        tot[n] += float(r[vi].replace(",", ""))
        cnt[n] += 1
    total = sum(tot.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for n in order:
        print(f"| `{n}` | {cnt[n]} | {tot[n] / cnt[n] / 1e3:.1f} | {tot[n] / 1e3:.1f} | {100 * tot[n] / total:.1f}% |")


def full(path, algo=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    algo = json.load(open(algo)) if algo else {}
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " | stall top-3 |")
    print("|---|" + "---|" * (len(KEYS) + 1))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        cells = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print(f"| `{name}` | " + " | ".join(cells) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in st[:3]) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
