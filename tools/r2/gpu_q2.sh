# deferred-factor rotations + diagonal regroup: new tests, full suite, cfg3/cfg4 A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tan.py -x -q -p no:cacheprovider > gpurun_out/q2_tan.log 2>&1
tail -5 gpurun_out/q2_tan.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --config 2 --steps 3 > gpurun_out/q2_c3.log 2>&1
TCX_NO_TAN=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q2_c3_notan.log 2>&1
TCX_NO_TAN=1 TCX_NO_DIAG_REGROUP=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q2_c3_none.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/q2_c4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/q2_tests.log 2>&1
tail -5 gpurun_out/q2_tests.log
for f in gpurun_out/q2_c*.log; do echo "== $f"; tail -1 $f | cut -c1-300; done
