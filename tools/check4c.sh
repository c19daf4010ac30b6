#!/bin/bash
# 4-GPU probes (under gpurun --gpus 4): copy-engine vs SM all-to-all NVLink at D=4 and D=3,
# e2e NUMA-binding A/B at N=2 and N=4.
tag=${1:-r01}
o=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_bench tools/p2p_bench.cu
timeout 300 tools/p2p_bench 4 512 > $o/${tag}_p2p_D4.json 2>&1; echo "p2p4 exit $?"
timeout 300 tools/p2p_bench 3 512 > $o/${tag}_p2p_D3.json 2>&1; echo "p2p3 exit $?"
for n in 2 4; do
  for v in 1 0; do
    LAMB_BENCH_NUMA=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29553 bench.py --gpus $n --steps 10 > $o/${tag}_e2e_n${n}_numa$v.log 2>&1; echo "bench n=$n numa=$v exit $?"
  done
done
nvidia-smi topo -m > $o/${tag}_topo.txt 2>&1
cat $o/${tag}_p2p_D4.json
