"""Write per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the pass
kernels from an ncu --set full report into profiles/ncu_traffic.json, keyed
"<workload>/D<world>/<comm>/<pass_a|pass_b>" (bench.py reads it for roofline.traffic).

    python tools/ncu_traffic.py <report.ncu-rep> <workload> <world> <comm>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, wl, D, comm = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
out = json.load(open(path)) if os.path.exists(path) else {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    key = "pass_a" if name.startswith("void pass_a") else "pass_b" if name.startswith("void pass_b") else None
    if not key:
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        b += float(r[i].replace(",", "")) * scale[units[i]]
    out[f"{wl}/D{D}/{comm}/{key}"] = {"bytes": b, "kernel": name.split("(")[0], "report": os.path.basename(rep)}
json.dump(out, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))
