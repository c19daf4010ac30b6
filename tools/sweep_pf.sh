#!/bin/bash
# pass A prefetch variants at D = 2 and 4 (fused): tools/sweep_pf.sh <out>
out=$1; : > $out
for n in 2 4; do
for t in "ua=4,ma=2,ub=4,mb=2,pf=0,upf=2" "ua=4,ma=2,ub=4,mb=2,pf=1,upf=2" "ua=4,ma=2,ub=4,mb=2,pf=1,upf=4"; do
  echo "{\"tune\": \"$t n=$n\"}" >> $out
  LAMB_TUNE=$t timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29561 bench.py --gpus $n --config 175b_slice_3l --steps 10 --warmup 3 --no-e2e >> $out 2>/dev/null
done; done
