#!/bin/bash
# 1-GPU box: the whole GPU suite, smoke, the bench, the ncu launch list of the bench command and
# one ncu --set full capture of the pass kernels (N = 1).  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
if [ "${SUITE:-1}" = 1 ]; then
  timeout 2700 python3 -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r02/pytest_gpu${TAG:-}.log 2>&1
  echo "pytest exit $?" >> gpurun_out/r02/pytest_gpu${TAG:-}.log
  grep -E "passed|failed|FAILED|ERROR" gpurun_out/r02/pytest_gpu${TAG:-}.log | tail -8
  python3 -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke${TAG:-}.log 2>&1; tail -1 gpurun_out/r02/smoke${TAG:-}.log
fi
timeout 900 python3 bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_n1${TAG:-}.json 2> gpurun_out/r02/bench_n1${TAG:-}.err
echo "bench exit $?"; tail -c 200 gpurun_out/r02/bench_n1${TAG:-}.json
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_n1.csv \
    python3 bench.py --steps 2 --warmup 3 --no-e2e --no-curve --no-cpu-baseline > gpurun_out/r02/ncu_launches.log 2>&1
  echo "ncu launches exit $?"
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'pass_[ab]' --launch-skip 6 -c 2 \
    -o gpurun_out/r02/full_n1 python3 bench.py --steps 2 --warmup 3 --no-e2e --no-curve --no-cpu-baseline > gpurun_out/r02/ncu_full.log 2>&1
  echo "ncu full exit $?"
fi
