#!/bin/bash
# Round-2 GPU check (1 GPU): build, the full GPU suite (incl. the 8-rank oversubscribed run),
# the pass-B mutants, a short bench.  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/r02/build.log; exit 1; }
timeout 2400 python3 -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_gpu.log
tail -3 gpurun_out/r02/pytest_gpu.log
if [ "${MUTANTS:-1}" = 1 ]; then
  bash tools/mutant_check.sh > gpurun_out/r02/mutants.log 2>&1
  cat gpurun_out/r02/mutants.log
fi
timeout 600 python3 bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_n1.json 2> gpurun_out/r02/bench_n1.err
tail -c 600 gpurun_out/r02/bench_n1.json
