#!/bin/bash
# Round-2 GPU check (1 GPU): build, the whole GPU suite without -x (every failure listed), a short
# bench.  Output under gpurun_out/r02/.
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/r02/build.log; exit 1; }
timeout 2700 python3 -m pytest tests -m gpu -q -s -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/r02/pytest_gpu${TAG:-}.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_gpu${TAG:-}.log
grep -E "passed|failed|FAILED|ERROR" gpurun_out/r02/pytest_gpu${TAG:-}.log | tail -20
python3 -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke${TAG:-}.log 2>&1; tail -2 gpurun_out/r02/smoke${TAG:-}.log
