#!/bin/bash
# 4-GPU box: the large BASELINE configs at D = 4 with the round-2 code (13B, 175B slice 12L,
# 530B slice + 32,768 stress tensors) and 13B at D = 2.  One JSON line each.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || exit 1
for cfg in gpt13b 175b_slice 530b_stress; do
  timeout 900 python3 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-curve --no-cpu-baseline >> gpurun_out/r02/big_n4.jsonl 2>> gpurun_out/r02/big_n4.err
  echo "$cfg exit $?"
done
timeout 900 python3 bench.py --gpus 2 --config gpt13b --steps 10 --warmup 3 --no-e2e --no-curve --no-cpu-baseline >> gpurun_out/r02/big_n4.jsonl 2>> gpurun_out/r02/big_n4.err
python3 - <<'PY'
import json
for l in open("gpurun_out/r02/big_n4.jsonl"):
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"], d["n_gpus"], round(d["ms_per_step"], 2), round(d["value"] / 1e9, 1), r["bound"], round(r["frac"], 3),
          (r.get("alltoall_ceiling") or {}).get("frac"))
PY
