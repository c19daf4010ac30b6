#!/bin/bash
# 2-GPU check (under gpurun --gpus 2): per-bucket lamb_step_host pipeline tests, e2e A/B
# (per-bucket vs whole-step pipeline) at N=1 and N=2, straddler hiding A/B at N=2.
tag=${1:-r01}
o=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "step_host" > $o/${tag}_pytest_host.log 2>&1; echo "pytest1 exit $?" >> $o/${tag}_pytest_host.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s -k "2gpu and fused" >> $o/${tag}_pytest_host.log 2>&1; echo "pytest2 exit $?" >> $o/${tag}_pytest_host.log
for v in 0 1; do
  LAMB_HOST_WHOLE=$v timeout 600 python bench.py --no-cpu-baseline > $o/${tag}_bench1_whole$v.log 2>&1; echo "bench1 whole=$v exit $?"
done
for v in 0 1 0 1; do
  LAMB_NO_STRAD_HIDE=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29551 bench.py --gpus 2 --no-e2e > $o/${tag}_bench2_nohide$v.log 2>&1; echo "bench2 nohide=$v exit $?"
  tail -1 $o/${tag}_bench2_nohide$v.log >> $o/${tag}_bench2_hide.jsonl
done
for v in 0 1; do
  LAMB_HOST_WHOLE=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29552 bench.py --gpus 2 > $o/${tag}_bench2_whole$v.log 2>&1; echo "bench2 whole=$v exit $?"
done
tail -3 $o/${tag}_pytest_host.log
