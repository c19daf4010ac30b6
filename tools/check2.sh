#!/bin/bash
# 2-GPU check (under gpurun --gpus 2): multi-GPU parity incl. the 8-rank oversubscribed case,
# straddler hiding A/B on the bench, host-link and NVLink probes.  Usage: tools/check2.sh <tag>
tag=${1:-r01}
o=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -s -k "2gpu or oversub" > $o/${tag}_pytest_multi2.log 2>&1; echo "pytest exit $?" >> $o/${tag}_pytest_multi2.log
for v in "" 1 "" 1; do
  LAMB_NO_STRAD_HIDE=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29551 bench.py --gpus 2 --no-e2e > $o/${tag}_bench2_hide$v.log 2>&1; echo "bench hide=$v exit $?"
  tail -1 $o/${tag}_bench2_hide$v.log >> $o/${tag}_bench2_hide.jsonl
done
timeout 300 python tools/pcie_probe.py > $o/${tag}_pcie.jsonl 2>&1; echo "pcie exit $?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_bench tools/p2p_bench.cu && timeout 300 tools/p2p_bench 2 512 > $o/${tag}_p2p_D2.json 2>&1; echo "p2p exit $?"
tail -3 $o/${tag}_pytest_multi2.log
