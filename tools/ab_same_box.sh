#!/bin/bash
# A/B on one box: the current tree vs an older build in _ab_old/ (bench, alternating), N=1 and N=2.
o=gpurun_out
: > $o/ab.jsonl
for rep in 1 2 3; do
  for d in . _ab_old; do
    echo "{\"tree\": \"$d n=1\"}" >> $o/ab.jsonl
    (cd $d && timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | tail -1) >> $o/ab.jsonl
    echo "{\"tree\": \"$d n=2\"}" >> $o/ab.jsonl
    (cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29560 bench.py --gpus 2 --no-e2e --steps 30 2>/dev/null | tail -1) >> $o/ab.jsonl
  done
done
