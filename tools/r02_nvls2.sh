#!/bin/bash
# 2-GPU box: NVLS mode parity (variant oracle) + the 2-GPU parity of FUSED/NCCL, then a same-box
# A/B of the step in FUSED vs NVLS mode.  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/r02/build.log; exit 1; }
timeout 1500 python3 -m pytest tests/test_gpu_multi.py -q -s -p no:cacheprovider -k "${PYK:-2gpu}" > gpurun_out/r02/pytest_multi2${TAG:-}.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_multi2${TAG:-}.log
grep -E "^\[ok\]|passed|failed|Error|error" gpurun_out/r02/pytest_multi2${TAG:-}.log | head -60
for c in fused nvls fused nvls; do
  timeout 600 python3 bench.py --gpus 2 --comm $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-curve >> gpurun_out/r02/ab_nvls_n2${TAG:-}.jsonl 2>> gpurun_out/r02/ab_nvls_n2${TAG:-}.err
done
python3 - <<'PY'
import json
import os
for l in open("gpurun_out/r02/ab_nvls_n2" + os.environ.get("TAG", "") + ".jsonl"):
    d = json.loads(l); p = d["phases_ms"]
    print(d["config"]["comm"], round(d["ms_per_step"], 3), "A", round(p["pass_a"], 3), "B", round(p["pass_b"], 3))
PY
