#!/bin/bash
# Scaling / large-config runs on one box (fused mode unless stated).  JSON lines -> $out.
# Usage (under gpurun --gpus 4): tools/scaling.sh gpurun_out/scaling_r01.jsonl
out=${1:-gpurun_out/scaling.jsonl}
: > $out
run() {  # n config extra...
  n=$1; cfg=$2; shift 2
  echo "{\"run\": \"n=$n $cfg $*\"}" >> $out
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --gpus 1 --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" >> $out 2>$out.err.$n.$cfg
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29540 bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-e2e "$@" >> $out 2>$out.err.$n.$cfg
  fi
  echo "rc=$? n=$n $cfg $*"
}
for n in 1 2 4; do run $n 175b_slice_3l; done
run 4 175b_slice_3l --comm nccl
for n in 2 4; do run $n gpt13b; done
run 4 175b_slice
run 4 530b_stress
