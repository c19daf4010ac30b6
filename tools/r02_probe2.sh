#!/bin/bash
# 2-GPU box: NVSwitch rounding probe of multimem.ld_reduce (reading Z23) and the ncu NVLink-byte
# captures of the fused passes (FUSED and NVLS, D = 2).
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { echo build failed; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_round_probe tools/nvls_round_probe.cu -lcuda && \
  timeout 300 /tmp/nvls_round_probe 2 gpurun_out/r02/nvls_round_D2.bin
bash tools/ncu_nvlink.sh fused 2
bash tools/ncu_nvlink.sh nvls 2
