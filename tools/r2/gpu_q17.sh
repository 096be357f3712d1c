# multi-box TMA windows: parity subset + A/B (cfg3, cfg2, cfg4, cfg5)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_shard.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/q17_tests.log 2>&1
tail -3 gpurun_out/q17_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --config 2 --steps 3 > gpurun_out/q17_c3.log 2>&1
TCX_TMA_NO_MULTIBOX=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q17_c3_off.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/q17_c2.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/q17_c4.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/q17_c5.log 2>&1
for f in gpurun_out/q17_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
