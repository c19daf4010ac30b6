"""NVLink bytes (nvlrx__bytes / nvltx__bytes, and their user-data parts; ncu, 32 B granularity)
and DRAM bytes of the pass kernels per GPU per step — summed over a device's launches of the
pass (pass B runs as two launches when the straddler exchange hides under it), averaged over
devices — from the CSV of an ncu run of tools/nvlink_bytes_1proc.py (one step per device), into
profiles/ncu_nvlink.json keyed
"<workload>/D<world>/<comm>/<pass_a|pass_b>" (bench.py reports them as roofline.nvlink.traffic
when NVML has no NVLink byte counters — the case on this pool, profiles/r02/nvlink_probe.jsonl).

    python tools/ncu_nvlink_json.py <csv> <workload> <world> <comm>
"""
import csv
import json
import os
import sys
from collections import defaultdict

path_csv, wl, D, comm = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}
lines = [l for l in open(path_csv) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
iid, iname, idev, imet, iunit, ival = (hdr.index(k) for k in ("ID", "Kernel Name", "Device", "Metric Name",
                                                                  "Metric Unit", "Metric Value"))
per = defaultdict(dict)
names, devs = {}, {}
for r in rows[1:]:
    per[r[iid]][r[imet]] = float(r[ival].replace(",", "")) * scale.get(r[iunit], 1.0)
    names[r[iid]] = r[iname]
    devs[r[iid]] = r[idev]
acc = defaultdict(lambda: defaultdict(lambda: defaultdict(float)))   # pass -> device -> metric -> sum
kern = {}
nl = defaultdict(int)
for k, m in per.items():
    n = names[k]
    key = "pass_a" if "pass_a" in n else "pass_b" if "pass_b" in n else None
    if key:
        for met, v in m.items():
            acc[key][devs[k]][met] += v
        kern[key] = n.split("(")[0]
        nl[key] += 1
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_nvlink.json")
out = json.load(open(out_path)) if os.path.exists(out_path) else {}
for key, bydev in acc.items():
    nd = len(bydev)
    mean = defaultdict(float)
    for d in bydev.values():
        for met, v in d.items():
            mean[met] += v / nd
    out[f"{wl}/D{D}/{comm}/{key}"] = {
        "nvlink_rx_bytes": mean.get("nvlrx__bytes.sum"), "nvlink_tx_bytes": mean.get("nvltx__bytes.sum"),
        "nvlink_rx_user_bytes": mean.get("nvlrx__bytes_data_user.sum"),
        "nvlink_tx_user_bytes": mean.get("nvltx__bytes_data_user.sum"),
        "dram_bytes": mean.get("dram__bytes_read.sum", 0) + mean.get("dram__bytes_write.sum", 0),
        "per": "GPU per step (sum of the device's launches, mean over devices)", "devices": nd,
        "launches": nl[key], "kernel": kern[key], "source": os.path.basename(path_csv)}
json.dump(out, open(out_path, "w"), indent=1, sort_keys=True)
print(json.dumps({k: v for k, v in out.items() if k.startswith(f"{wl}/D{D}/{comm}/")}, indent=1))
