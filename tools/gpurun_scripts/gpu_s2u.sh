set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_noise.py tests/test_gpu_dense.py -x -q > gpurun_out/s2u_t.log 2>&1
tail -5 gpurun_out/s2u_t.log
timeout 600 python bench.py --config 5 --steps 50 > gpurun_out/s2u_t7.log 2>&1
tail -1 gpurun_out/s2u_t7.log | cut -c1-200
