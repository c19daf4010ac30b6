#!/bin/bash
# pass B bulk param stores (LAMB_TUNE tmb=1) vs STG (tmb=0) at N = 1, 2, 4 + parity with tmb=1.
o=gpurun_out
base="ua=4,ma=2,ub=4,mb=2,pf=1,upf=4,ring=0,tma=1,tmam=1,tmb="
LAMB_TUNE=${base}1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $o/tmb_pytest.log 2>&1; echo "pytest1 exit $?"
LAMB_TUNE=${base}1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k "4gpu and fused" >> $o/tmb_pytest.log 2>&1; echo "pytest4 exit $?"
: > $o/tmb_bench.jsonl
for rep in 1 2; do
  for v in 0 1; do
    echo "{\"tune\": \"n=1 tmb=$v\"}" >> $o/tmb_bench.jsonl
    LAMB_TUNE=${base}$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | tail -1 >> $o/tmb_bench.jsonl
    for n in 2 4; do
      echo "{\"tune\": \"n=$n tmb=$v\"}" >> $o/tmb_bench.jsonl
      LAMB_TUNE=${base}$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29555 bench.py --gpus $n --no-e2e --steps 20 2>/dev/null | tail -1 >> $o/tmb_bench.jsonl
    done
  done
done
grep -E "passed|failed" $o/tmb_pytest.log
