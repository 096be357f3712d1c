# backward tile pipeline revisited (t = 12 and t = 11) on cfg3 / cfg2
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
TCX_JIT_PIPE=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/q16_c3_p1.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 2 --steps 3 --tile-bits 11 > gpurun_out/q16_c3_p1_t11.log 2>&1
TCX_JIT_PIPE=1 TCX_JIT_MINB=2 timeout 600 $B --config 2 --steps 3 --tile-bits 11 > gpurun_out/q16_c3_p1_t11_m2.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --steps 5 > gpurun_out/q16_c2_p1.log 2>&1
for f in gpurun_out/q16_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
