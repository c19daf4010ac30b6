#!/bin/bash
# pass A ring variants (LAMB_TUNE tmam=1 single ring; 3: decoupled grad ring, state 2 deep;
# 4/5: own slice in the state ring (2/3 deep), remote slices in the deep ring) at N = 2 and 4.
o=gpurun_out
base="ua=4,ma=2,ub=4,mb=2,pf=1,upf=4,ring=0,tma=1,tmam="
LAMB_TUNE=${base}4 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k "2gpu and fused" > $o/tma2_pytest.log 2>&1; echo "pytest4 exit $?"
LAMB_TUNE=${base}5 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k "2gpu and fused" >> $o/tma2_pytest.log 2>&1; echo "pytest5 exit $?"
: > $o/tma2_bench.jsonl
for n in 2 4; do
  for rep in 1 2; do
    for v in 1 3 4 5; do
      if [ $n -eq 4 ] && [ $v -eq 5 ]; then continue; fi
      echo "{\"tune\": \"n=$n tmam=$v\"}" >> $o/tma2_bench.jsonl
      LAMB_TUNE=${base}$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29554 bench.py --gpus $n --no-e2e --steps 20 2>/dev/null | tail -1 >> $o/tma2_bench.jsonl
    done
  done
done
grep -E "passed|failed" $o/tma2_pytest.log
