# forward-only TMA pipeline A/B (cfg2, cfg3, cfg5)
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 600 $B --steps 5 > gpurun_out/q6_c2.log 2>&1
TCX_JIT_PIPE=2 timeout 600 $B --steps 5 > gpurun_out/q6_c2_p2.log 2>&1
timeout 600 $B --config 2 --steps 3 > gpurun_out/q6_c3.log 2>&1
TCX_JIT_PIPE=2 timeout 600 $B --config 2 --steps 3 > gpurun_out/q6_c3_p2.log 2>&1
TCX_JIT_PIPE=2 timeout 900 $B --config 4 --steps 3 > gpurun_out/q6_c5_p2.log 2>&1
TCX_JIT_PIPE=2 timeout 900 $B --config 3 --steps 2 > gpurun_out/q6_c4_p2.log 2>&1
for f in gpurun_out/q6_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
