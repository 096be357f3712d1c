# kind-3 (general runs) correctness + A/B; cfg3 pipeline / tile variants
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tan.py -q -p no:cacheprovider > gpurun_out/q5_tan.log 2>&1
tail -5 gpurun_out/q5_tan.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --steps 5 > gpurun_out/q5_c2.log 2>&1
TCX_NO_TAN=1 timeout 600 $B --steps 5 > gpurun_out/q5_c2_notan.log 2>&1
timeout 300 $B --config 0 --steps 50 > gpurun_out/q5_c1.log 2>&1
TCX_NO_TAN=1 timeout 300 $B --config 0 --steps 50 > gpurun_out/q5_c1_notan.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q5_c3_pipe.log 2>&1
timeout 600 $B --config 2 --steps 3 --tile-bits 13 --coalesce-bits 2 > gpurun_out/q5_c3_t13.log 2>&1
timeout 600 $B --config 2 --steps 3 --reg-bits 3 > gpurun_out/q5_c3_r3.log 2>&1
for f in gpurun_out/q5_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
