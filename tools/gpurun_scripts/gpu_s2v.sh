set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/s2v_fuzz.log 2>&1
tail -15 gpurun_out/s2v_fuzz.log
