#!/bin/bash
# 4-GPU box: TMA pull all-to-all ceiling, NVSwitch rounding at D = 4, NVLS parity at D = 4, the
# FUSED vs NVLS A/B at D = 4 and the default bench at N = 4 (self-launched, with the 175B-3L curve
# point).  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p_bench tools/p2p_bench.cu && \
  for D in 4 2; do timeout 300 /tmp/p2p_bench $D 256 1 >> gpurun_out/r02/p2p_tma_pull.jsonl; done
tail -2 gpurun_out/r02/p2p_tma_pull.jsonl
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_round_probe tools/nvls_round_probe.cu -lcuda && \
  timeout 300 /tmp/nvls_round_probe 4 gpurun_out/r02/nvls_round_D4.bin
timeout 1500 python3 -m pytest tests/test_gpu_multi.py -q -s -p no:cacheprovider -k "4gpu_nvls" > gpurun_out/r02/pytest_multi4_nvls.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_multi4_nvls.log
grep -E "^\[ok\]|passed|failed|Error" gpurun_out/r02/pytest_multi4_nvls.log | head -30
for c in fused nvls fused nvls; do
  timeout 600 python3 bench.py --gpus 4 --comm $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-curve >> gpurun_out/r02/ab_nvls_n4.jsonl 2>> gpurun_out/r02/ab_nvls_n4.err
done
python3 - <<'PY'
import json
for l in open("gpurun_out/r02/ab_nvls_n4.jsonl"):
    d = json.loads(l); p = d["phases_ms"]
    print(d["config"]["comm"], round(d["ms_per_step"], 3), "A", round(p["pass_a"], 3), "B", round(p["pass_b"], 3))
PY
timeout 900 python3 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02/bench_n4.json 2> gpurun_out/r02/bench_n4.err
tail -c 300 gpurun_out/r02/bench_n4.json
