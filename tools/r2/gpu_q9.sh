# CNOT external controls as selects vs uniform branches (cfg2, cfg1, cfg5)
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 600 $B --steps 5 > gpurun_out/q9_c2.log 2>&1
TCX_JIT_CX_SEL=1 timeout 600 $B --steps 5 > gpurun_out/q9_c2_sel.log 2>&1
TCX_JIT_CX_SEL=1 timeout 300 $B --config 0 --steps 50 > gpurun_out/q9_c1_sel.log 2>&1
TCX_JIT_CX_SEL=1 timeout 900 $B --config 4 --steps 3 > gpurun_out/q9_c5_sel.log 2>&1
for f in gpurun_out/q9_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
