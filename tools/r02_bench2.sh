#!/bin/bash
# 2-GPU box: NVLink counter probe, the bench at N=1 (with the curve point and the CPU legs) and
# N=2 (self-launched), the bench contract tests.  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/r02/build.log; exit 1; }
nvidia-smi topo -m > gpurun_out/r02/topo.txt 2>&1
timeout 300 python3 tools/nvlink_counter_probe.py > gpurun_out/r02/nvlink_probe.jsonl 2> gpurun_out/r02/nvlink_probe.err
timeout 900 python3 bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_n1${TAG:-}.json 2> gpurun_out/r02/bench_n1${TAG:-}.err
tail -c 400 gpurun_out/r02/bench_n1${TAG:-}.json
timeout 900 python3 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02/bench_n2${TAG:-}.json 2> gpurun_out/r02/bench_n2${TAG:-}.err
tail -c 400 gpurun_out/r02/bench_n2${TAG:-}.json
timeout 1200 python3 -m pytest tests/test_gpu_bench.py -q -s -p no:cacheprovider > gpurun_out/r02/pytest_bench.log 2>&1
tail -3 gpurun_out/r02/pytest_bench.log
