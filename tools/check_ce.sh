#!/bin/bash
# copy-engine schedule: parity (D=2, D=8 oversubscribed) and the overlap harness at N=2 (and N=4 if present).
o=gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -s -k "2gpu and fused or oversub" > $o/ce_pytest.log 2>&1; echo "pytest exit $?"
grep -E "copy-engine|passed|failed|Error" $o/ce_pytest.log | head
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 \
  tools/bench_overlap.py --ctas 0 --green "" > $o/ce_overlap2.log 2>&1; echo "overlap2 exit $?"
if [ $N -ge 4 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29559 \
  tools/bench_overlap.py --ctas 0 --green "" > $o/ce_overlap4.log 2>&1; echo "overlap4 exit $?"
fi
tail -1 $o/ce_overlap2.log
