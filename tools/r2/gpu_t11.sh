# two-deep prefetch ring for forward passes (TCX_JIT_PIPE_DEPTH=2): parity + A/B
set -x
mkdir -p gpurun_out/t11
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t11cache
TCX_JIT_PIPE_DEPTH=2 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_gpu_inputs.py -q -x -p no:cacheprovider > gpurun_out/t11/tests.log 2>&1
tail -3 gpurun_out/t11/tests.log
timeout 600 $B --config 2 --steps 3 > gpurun_out/t11/c3.log 2>&1
TCX_JIT_PIPE_DEPTH=2 timeout 600 $B --config 2 --steps 3 > gpurun_out/t11/c3_d2.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t11/c2.log 2>&1
TCX_JIT_PIPE_DEPTH=2 timeout 600 $B --steps 5 > gpurun_out/t11/c2_d2.log 2>&1
timeout 600 $B --config 1 --max-ops-per-pass 1 --steps 2 > gpurun_out/t11/pg.log 2>&1
TCX_JIT_PIPE_DEPTH=2 timeout 600 $B --config 1 --max-ops-per-pass 1 --steps 2 > gpurun_out/t11/pg_d2.log 2>&1
TCX_JIT_PIPE_DEPTH=2 timeout 900 $B --config 3 --steps 2 > gpurun_out/t11/c4_d2.log 2>&1
TCX_JIT_PIPE_DEPTH=2 timeout 900 $B --config 4 --steps 3 > gpurun_out/t11/c5_d2.log 2>&1
for f in gpurun_out/t11/*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
