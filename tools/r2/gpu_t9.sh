# L2 prefetch of the next tile's lambda in half-pipelined passes (TCX_JIT_LAMPF) and multi-box TMA
# tiles for scattered windows (TCX_TMA_MULTIBOX) under the session-3 defaults
set -x
mkdir -p gpurun_out/t9
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t9cache
timeout 600 $B --config 2 --steps 3 > gpurun_out/t9/c3.log 2>&1
TCX_JIT_LAMPF=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t9/c3_lampf.log 2>&1
TCX_TMA_MULTIBOX=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t9/c3_mb.log 2>&1
TCX_TMA_MULTIBOX=1 TCX_JIT_LAMPF=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t9/c3_mb_lampf.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t9/c2.log 2>&1
TCX_JIT_LAMPF=1 timeout 600 $B --steps 5 > gpurun_out/t9/c2_lampf.log 2>&1
TCX_JIT_LAMPF=1 timeout 900 $B --config 4 --steps 3 > gpurun_out/t9/c5_lampf.log 2>&1
for f in gpurun_out/t9/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
TCX_JIT_LAMPF=1 TCX_TMA_MULTIBOX=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py -q -x -p no:cacheprovider > gpurun_out/t9/tests.log 2>&1
tail -3 gpurun_out/t9/tests.log
