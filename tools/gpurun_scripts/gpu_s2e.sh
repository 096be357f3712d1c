set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_terms.py tests/test_gpu_inputs.py -x -q > gpurun_out/s2e_t.log 2>&1
tail -15 gpurun_out/s2e_t.log
