#!/bin/bash
# One-GPU evidence run: parity tests, the default bench line, the ncu launch list of the same
# bench command, and one ncu --set full capture of pass A / finalize / pass B (step 2).
# Usage (under gpurun): tools/profile_n1.sh <tag>
tag=${1:-r01}
o=gpurun_out
python -m pytest tests -m gpu -x -q > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $o/${tag}_pytest_gpu.log
python bench.py > $o/${tag}_bench.log 2>&1; echo "bench exit $?"
B="bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
python $B > $o/${tag}_b_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches.csv python $B > $o/${tag}_ncu_launch.log 2>&1
P="tools/prof_step.py --steps 2"
python $P > $o/${tag}_prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"pass_a|pass_b|finalize" -s 3 -c 3 -o $o/${tag}_full python $P > $o/${tag}_ncu_full.log 2>&1
tail -2 $o/${tag}_pytest_gpu.log; tail -1 $o/${tag}_bench.log | cut -c1-400; ls $o
