#!/bin/bash
# ONE compute-sanitizer tool per gpurun call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || exit 1
timeout 300 python3 tools/sanitize_toy.py > gpurun_out/r02/sanitize_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool $TOOL --kernel-name kre=lamb --error-exitcode 9 python3 tools/sanitize_toy.py \
   > gpurun_out/r02/sanitize_$TOOL.log 2>&1
echo "sanitizer $TOOL exit $?"
tail -6 gpurun_out/r02/sanitize_$TOOL.log
