set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q -k "dpsi or grad" > gpurun_out/s2s_t.log 2>&1
tail -5 gpurun_out/s2s_t.log
timeout 600 python bench.py --config 0 --steps 50 --no-cpu-baseline > gpurun_out/s2s_c1.log 2>&1
tail -1 gpurun_out/s2s_c1.log | cut -c1-150
