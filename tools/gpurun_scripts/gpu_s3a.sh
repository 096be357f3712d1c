set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_noise.py tests/test_gpu_fuzz.py tests/test_gpu_inputs.py -x -q > gpurun_out/s3a_t.log 2>&1
tail -3 gpurun_out/s3a_t.log
timeout 900 python bench.py --config 1 --dense-k 2 --steps 2 --no-cpu-baseline > gpurun_out/s3a_c2k2.log 2>&1
tail -1 gpurun_out/s3a_c2k2.log | cut -c1-150
