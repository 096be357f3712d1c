set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2k_t.log 2>&1
tail -3 gpurun_out/s2k_t.log
