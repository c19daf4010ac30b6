mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi topo -m; cat /proc/meminfo | head -3; df -h /dev/shm) > gpurun_out/box_info.txt 2>&1
timeout 300 python tools/nvlink_counter_probe.py > gpurun_out/nvlink_probe.jsonl 2> gpurun_out/nvlink_probe.err
echo done
