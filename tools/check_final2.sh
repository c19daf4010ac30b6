#!/bin/bash
# 2-GPU closing checks: smoke(), the reference arm, graph-mode bench, soak at D=1 (graph) and D=2.
o=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/fin_smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/fin_ref.log 2>&1; echo "ref exit $?"
timeout 600 python bench.py --graph --no-e2e --no-cpu-baseline > $o/fin_graph1.log 2>&1; echo "graph1 exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 \
  bench.py --gpus 2 --graph --no-e2e > $o/fin_graph2.log 2>&1; echo "graph2 exit $?"
timeout 900 python tests/soak.py --steps 2000 --graph > $o/fin_soak1g.json 2>&1; echo "soak1 exit $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 \
  tests/soak.py --steps 2000 > $o/fin_soak2.json 2>&1; echo "soak2 exit $?"
tail -2 $o/fin_smoke.log
