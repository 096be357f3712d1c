# batched gradient reductions: parity subset + rbatch A/B on cfg3 / cfg2
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tan.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/q8_tests.log 2>&1
tail -3 gpurun_out/q8_tests.log
B="python bench.py --no-cpu-baseline"
for rb in 1 4 8; do
  TCX_JIT_RBATCH=$rb timeout 600 $B --config 2 --steps 3 > gpurun_out/q8_c3_rb$rb.log 2>&1
done
timeout 600 $B --steps 5 > gpurun_out/q8_c2.log 2>&1
for f in gpurun_out/q8_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
