#!/bin/bash
# D-GPU box: per-kernel NVLink (and DRAM) bytes of the FUSED passes with ncu on ONE process driving
# the D GPUs (tools/nvlink_bytes_1proc.py).  ncu cannot profile the multimem (NVLS) kernels
# ("UnknownError", r02).  Output: gpurun_out/r02/ncu_nvlink_fused_D<D>_gpt1.3b.csv
set -u
mkdir -p gpurun_out/r02
python3 -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || exit 1
for D in ${DS:-2}; do
  timeout 600 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:'pass_[ab]' --csv --log-file gpurun_out/r02/ncu_nvlink_fused_D${D}_gpt1.3b.csv \
    python3 tools/nvlink_bytes_1proc.py $D fused gpt1.3b > gpurun_out/r02/nvl1p_fused_D$D.log 2>&1
  echo "ncu D=$D exit $?"; tail -2 gpurun_out/r02/nvl1p_fused_D$D.log
done
