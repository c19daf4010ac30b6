#!/bin/bash
# NVLink bytes of the fused passes, measured: rank 0 of a D-rank bench runs under ncu with the
# per-kernel NVLink counters (nvlrx__bytes / nvltx__bytes, 32 B granularity) next to DRAM bytes
# and duration; the other ranks run plainly (their barriers wait, LAMB_BARRIER_TIMEOUT_MS raised).
# Times under ncu are serialised replays: only the BYTES are used.
#   bash tools/ncu_nvlink.sh <fused|nvls> <D> [config]      -> gpurun_out/r02/ncu_nvlink_<comm>_D<D>.csv
set -u
COMM=$1; D=$2; CFG=${3:-gpt1.3b}
mkdir -p gpurun_out/r02
OUT=gpurun_out/r02/ncu_nvlink_${COMM}_D${D}_${CFG}.csv
W=/tmp/lamb_rankwrap_$$.sh
cat > $W <<EOS
#!/bin/bash
ARGS="bench.py --gpus $D --comm $COMM --config $CFG --steps 3 --warmup 3 --no-e2e --no-curve --no-cpu-baseline"
if [ "\$RANK" = "0" ]; then
  exec ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:'pass_[ab]' --launch-skip 2 -c 4 --csv --log-file $OUT python3 \$ARGS
else
  exec python3 \$ARGS
fi
EOS
chmod +x $W
LAMB_BARRIER_TIMEOUT_MS=900000 timeout 1500 python3 -m torch.distributed.run --nnodes=1 --nproc-per-node $D \
    --master-addr 127.0.0.1 --master-port 29555 --no-python bash $W > gpurun_out/r02/ncu_nvlink_${COMM}_D${D}.log 2>&1
echo "ncu run exit $?"
grep -E "pass_|nvl" $OUT | head -40
