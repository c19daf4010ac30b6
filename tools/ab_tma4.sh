#!/bin/bash
# D=1 pass A: 3-stage (tma=1) vs 4-stage (tma=2) TMA ring, alternating, plus a parity subset.
o=gpurun_out
base="ua=4,ma=2,ub=4,mb=2,pf=1,upf=4,ring=0,tma="
LAMB_TUNE=${base}2 timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "toy or determinism or ragged" > $o/tma4_pytest.log 2>&1; echo "pytest exit $?"; tail -1 $o/tma4_pytest.log
: > $o/tma4.jsonl
for v in 1 2 1 2; do
  echo "{\"tma\": $v}" >> $o/tma4.jsonl
  LAMB_TUNE=${base}$v timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | tail -1 >> $o/tma4.jsonl
done
