set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q -k "dpsi" > gpurun_out/s2w_tq.log 2>&1
tail -15 gpurun_out/s2w_tq.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2w_t.log 2>&1
tail -3 gpurun_out/s2w_t.log
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2w_c2.log 2>&1
tail -1 gpurun_out/s2w_c2.log | cut -c1-120
