set -x
mkdir -p gpurun_out
TCX_JIT_DBUF=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/s2x_t.log 2>&1
tail -3 gpurun_out/s2x_t.log
TCX_JIT_DBUF=1 timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2x_c2_dbuf.log 2>&1
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2x_c2.log 2>&1
TCX_JIT_DBUF=1 timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s2x_c3_dbuf.log 2>&1
TCX_JIT_DBUF=1 timeout 900 python bench.py --config 0 --steps 50 --no-cpu-baseline > gpurun_out/s2x_c1_dbuf.log 2>&1
for f in gpurun_out/s2x_c*.log; do echo $f; tail -1 $f | cut -c1-120; done
