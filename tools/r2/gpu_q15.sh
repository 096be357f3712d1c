# stage lookahead (K = 4) vs greedy: parity subset + cfg1 / cfg2 / cfg4 / cfg5
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -q -x -p no:cacheprovider > gpurun_out/q15_tests.log 2>&1
tail -3 gpurun_out/q15_tests.log
B="python bench.py --no-cpu-baseline"
timeout 300 $B --config 0 --steps 50 > gpurun_out/q15_c1.log 2>&1
TCX_STAGE_LOOKAHEAD=0 timeout 300 $B --config 0 --steps 50 > gpurun_out/q15_c1_g.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/q15_c2.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/q15_c4.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/q15_c5.log 2>&1
for f in gpurun_out/q15_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
