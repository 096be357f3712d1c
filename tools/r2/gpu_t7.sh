# lambda-unit windows with 64-byte runs under 32-byte-run plans (cfg5), new tests, parity subset
set -x
mkdir -p gpurun_out/t7
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t7cache
timeout 900 $B --config 4 --steps 3 > gpurun_out/t7/c5.log 2>&1
TCX_LAM_SAME_C=1 timeout 900 $B --config 4 --steps 3 > gpurun_out/t7/c5_samec.log 2>&1
timeout 600 $B --steps 5 --coalesce-bits 2 > gpurun_out/t7/c2_cb2.log 2>&1
for f in gpurun_out/t7/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
timeout 2400 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_terms.py tests/test_gpu_inputs.py tests/test_gpu_large.py tests/test_gpu_noise.py -q -x -p no:cacheprovider > gpurun_out/t7/tests.log 2>&1
tail -3 gpurun_out/t7/tests.log
