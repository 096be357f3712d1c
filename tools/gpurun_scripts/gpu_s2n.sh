set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_noise.py -x -q > gpurun_out/s2n_tnoise.log 2>&1
tail -15 gpurun_out/s2n_tnoise.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2n_t.log 2>&1
tail -3 gpurun_out/s2n_t.log
