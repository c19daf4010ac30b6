#!/bin/bash
# fused multi-GPU TMA passes on/off at N=2,4 (1.3B): tools/sweep_tma.sh <out>
out=$1; : > $out
for n in 2 4; do
for m in 0 1; do
  t="ua=4,ma=2,ub=4,mb=2,pf=1,upf=4,ring=0,tma=1,tmam=$m"
  echo "{\"tune\": \"$t n=$n\"}" >> $out
  LAMB_TUNE=$t timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29641 bench.py --gpus $n --steps 30 --warmup 3 --no-e2e >> $out 2>/dev/null
done; done
