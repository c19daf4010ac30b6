#!/bin/bash
# 1-GPU box: the LAMB_DEBUG build's GPU tests (checks fire on corruption; silent on the parity suite
# and the 8-rank oversubscribed protocol).
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; tail -5 gpurun_out/r02/build.log; exit 1; }
timeout 2400 python3 -m pytest tests/test_gpu_debug.py -q -s -p no:cacheprovider ${PYK:+-k "$PYK"} > gpurun_out/r02/pytest_debug.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02/pytest_debug.log
grep -E "passed|failed|LAMB_DEBUG|Error" gpurun_out/r02/pytest_debug.log | head -20
