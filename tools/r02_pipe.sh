#!/bin/bash
# D-GPU box (D = 2 or 4): the pipelined schedule — parity (FUSED bitwise vs plain, NVLS against
# the oracle) and a same-box A/B of FUSED / NVLS, plain / pipelined with K chunks.
set -u
D=${D:-4}
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python3 -m pytest tests/test_gpu_multi.py -q -s -p no:cacheprovider -k "${PYK:-${D}gpu_nvls or ${D}gpu and fused}" > gpurun_out/r02/pytest_pipe_n$D.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_pipe_n$D.log
grep -E "^\[ok\]|passed|failed|Error" gpurun_out/r02/pytest_pipe_n$D.log | head -60
for rep in 1 2; do
for cfg in "fused 0" "fused 4" "nvls 0" "nvls 4" "nvls 8" "fused 8"; do
  set -- $cfg
  timeout 600 python3 bench.py --gpus $D --comm $1 --pipe $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-curve >> gpurun_out/r02/ab_pipe_n$D.jsonl 2>> gpurun_out/r02/ab_pipe_n$D.err
done
done
python3 - <<PY
import json
for l in open("gpurun_out/r02/ab_pipe_n$D.jsonl"):
    d = json.loads(l); p = d["phases_ms"]
    print(d["config"]["comm"], d["config"].get("pipe"), round(d["ms_per_step"], 3), "A", round(p["pass_a"], 3), "B", round(p["pass_b"], 3))
PY
