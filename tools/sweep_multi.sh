#!/bin/bash
# LAMB_TUNE sweep of the fused multi-GPU kernels: tools/sweep_multi.sh <out> <n> <config>
out=$1; n=$2; cfg=$3
for t in "ua=4,ma=2,ub=4,mb=2" "ua=4,ma=3,ub=4,mb=3" "ua=2,ma=3,ub=2,mb=3" "ua=2,ma=4,ub=2,mb=4"; do
  echo "{\"tune\": \"$t n=$n $cfg\"}" >> $out
  LAMB_TUNE=$t timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29541 bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-e2e >> $out 2>/dev/null
done
