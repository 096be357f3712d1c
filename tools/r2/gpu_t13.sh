# lambda's TMA store as its own first bulk group in half-pipelined passes (TCX_JIT_LAMFIRST=1)
set -x
mkdir -p gpurun_out/t13
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t13cache
TCX_JIT_LAMFIRST=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py -q -x -p no:cacheprovider > gpurun_out/t13/tests.log 2>&1
tail -3 gpurun_out/t13/tests.log
timeout 600 $B --config 2 --steps 3 > gpurun_out/t13/c3.log 2>&1
TCX_JIT_LAMFIRST=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t13/c3_lf.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t13/c2.log 2>&1
TCX_JIT_LAMFIRST=1 timeout 600 $B --steps 5 > gpurun_out/t13/c2_lf.log 2>&1
TCX_JIT_LAMFIRST=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t13/c3_lf2.log 2>&1
timeout 600 $B --config 2 --steps 3 > gpurun_out/t13/c3_2.log 2>&1
for f in gpurun_out/t13/*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
