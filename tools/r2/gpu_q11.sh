# early cp.async next-tile loads for non-TMA backward windows: parity subset + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py -q -x -p no:cacheprovider -k "qaoa or cfg3 or tan or multi_pass or random" > gpurun_out/q11_tests.log 2>&1
tail -3 gpurun_out/q11_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --config 2 --steps 3 > gpurun_out/q11_c3.log 2>&1
TCX_JIT_EARLY_OFF=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q11_c3_off.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/q11_c4.log 2>&1
for f in gpurun_out/q11_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
