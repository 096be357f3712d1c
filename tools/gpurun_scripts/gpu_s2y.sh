set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "cfg4" > gpurun_out/s2y_t.log 2>&1
tail -5 gpurun_out/s2y_t.log
