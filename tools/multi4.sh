#!/bin/bash
# Multi-GPU evidence run on a 4-GPU box (under gpurun --gpus 4): every GPU test, the default bench
# line at N = 2 and 4, then the large-config scaling runs.  Usage: tools/multi4.sh <tag>
tag=${1:-r01}
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > $o/${tag}_pytest_gpu4.log 2>&1; echo "pytest exit $?" >> $o/${tag}_pytest_gpu4.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29550 bench.py --gpus $n > $o/${tag}_bench_n$n.log 2>&1; echo "bench n=$n exit $?"
done
bash tools/scaling.sh $o/${tag}_scaling.jsonl
tail -2 $o/${tag}_pytest_gpu4.log
