#!/bin/bash
# 4-GPU box: how the fused passes scale with the SM count (is a pass SM/latency-limited or
# fabric-limited?) — FUSED and NVLS at 148 / 74 / 37 CTAs.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || exit 1
for c in fused nvls; do for n in 148 74 37; do
  timeout 600 python3 bench.py --gpus 4 --comm $c --max-ctas $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-curve >> gpurun_out/r02/ctas_n4.jsonl 2>> gpurun_out/r02/ctas_n4.err
done; done
python3 - <<PY
import json
for l in open("gpurun_out/r02/ctas_n4.jsonl"):
    d = json.loads(l); p = d["phases_ms"]
    print(d["config"]["comm"], d["config"]["max_ctas"], round(d["ms_per_step"], 3), "A", round(p["pass_a"], 3), "B", round(p["pass_b"], 3))
PY
