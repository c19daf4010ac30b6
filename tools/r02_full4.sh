#!/bin/bash
# 4-GPU box, closing check of round 2: the whole GPU suite (every multi-GPU case at D = 2, 3, 4,
# FUSED / NCCL / NVLS, the full-size configs, the 8-rank oversubscribed run, the debug build,
# the bench contract incl. the self-launched 2-rank line), smoke, and bench lines at N = 1, 2, 4.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi topo -m > gpurun_out/r02/topo4.txt 2>&1
timeout 4000 python3 -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r02/pytest_gpu_4gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_gpu_4gpu.log
grep -E "passed|failed|FAILED|ERROR" gpurun_out/r02/pytest_gpu_4gpu.log | tail -12
python3 -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke4.log 2>&1; tail -1 gpurun_out/r02/smoke4.log
for n in 1 2 4; do
  timeout 900 python3 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02/bench_final_n$n.json 2> gpurun_out/r02/bench_final_n$n.err
  echo "bench n=$n exit $?"; tail -c 150 gpurun_out/r02/bench_final_n$n.json
done
