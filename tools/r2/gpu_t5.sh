# new defaults (interleaved tiles when a row's CTAs are co-resident, half pipeline on) +
# coalesce-bits sweep per config; parity subset under the new defaults
set -x
mkdir -p gpurun_out/t5
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t5cache
timeout 600 $B --config 2 --steps 3 > gpurun_out/t5/c3.log 2>&1
timeout 600 $B --config 2 --steps 3 --coalesce-bits 2 > gpurun_out/t5/c3_cb2.log 2>&1
timeout 600 $B --config 2 --steps 3 --coalesce-bits 4 > gpurun_out/t5/c3_cb4.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t5/c2.log 2>&1
timeout 600 $B --steps 5 --coalesce-bits 2 > gpurun_out/t5/c2_cb2.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/t5/c5.log 2>&1
timeout 900 $B --config 4 --steps 3 --coalesce-bits 2 > gpurun_out/t5/c5_cb2.log 2>&1
TCX_JIT_HALFPIPE=0 timeout 900 $B --config 4 --steps 3 --coalesce-bits 2 > gpurun_out/t5/c5_cb2_nohalf.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/t5/c4.log 2>&1
timeout 900 $B --config 3 --steps 2 --coalesce-bits 1 > gpurun_out/t5/c4_cb1.log 2>&1
for f in gpurun_out/t5/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_shard.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/t5/tests.log 2>&1
tail -3 gpurun_out/t5/tests.log
