# early next-tile TMA load in backward kernels: parity subset + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_shard.py -q -x -p no:cacheprovider > gpurun_out/q10_tests.log 2>&1
tail -3 gpurun_out/q10_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --steps 5 > gpurun_out/q10_c2.log 2>&1
TCX_JIT_EARLY_OFF=1 timeout 600 $B --steps 5 > gpurun_out/q10_c2_off.log 2>&1
timeout 600 $B --config 2 --steps 3 > gpurun_out/q10_c3.log 2>&1
TCX_JIT_EARLY_OFF=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q10_c3_off.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/q10_c5.log 2>&1
for f in gpurun_out/q10_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
