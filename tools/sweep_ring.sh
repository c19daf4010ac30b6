#!/bin/bash
# cp.async ring depth for the fused pass A at D=2: tools/sweep_ring.sh <out>
out=$1; : > $out
for r in 0 3 4 6; do
  t="ua=4,ma=2,ub=4,mb=2,pf=1,upf=4,ring=$r"
  echo "{\"tune\": \"$t\"}" >> $out
  LAMB_TUNE=$t timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29601 bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e >> $out 2>/dev/null
done
