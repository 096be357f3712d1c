set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/p1_smi.txt
free -g > gpurun_out/p1_host.txt; nproc >> gpurun_out/p1_host.txt; lscpu | grep -i "model name\|socket\|core" >> gpurun_out/p1_host.txt
timeout 900 python tools/r2/probe_n33.py > gpurun_out/p1_n33.log 2>&1
tail -20 gpurun_out/p1_n33.log
