# smaller tiles (t = 11: 128-thread CTAs, up to 4 per SM) for the ALU-bound headline and cfg3
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 900 $B --steps 5 --tile-bits 11 > gpurun_out/q13_c2_t11.log 2>&1
TCX_JIT_MINB=4 timeout 900 $B --steps 5 --tile-bits 11 > gpurun_out/q13_c2_t11_m4.log 2>&1
TCX_JIT_MINB=3 timeout 900 $B --steps 5 --tile-bits 11 > gpurun_out/q13_c2_t11_m3.log 2>&1
timeout 900 $B --steps 5 --tile-bits 11 --coalesce-bits 2 > gpurun_out/q13_c2_t11_c2.log 2>&1
TCX_JIT_MINB=4 timeout 900 $B --config 2 --steps 3 --tile-bits 11 > gpurun_out/q13_c3_t11_m4.log 2>&1
timeout 900 $B --config 2 --steps 3 --tile-bits 11 > gpurun_out/q13_c3_t11.log 2>&1
for f in gpurun_out/q13_c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
TCX_JIT_MINB_FWD=3 timeout 900 $B --config 2 --steps 3 > gpurun_out/q13_c3_fm3.log 2>&1
TCX_JIT_MINB_FWD=3 timeout 900 $B --steps 5 > gpurun_out/q13_c2_fm3.log 2>&1
TCX_JIT_MINB_FWD=3 timeout 900 $B --config 3 --steps 2 > gpurun_out/q13_c4_fm3.log 2>&1
for f in gpurun_out/q13_c*fm3.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
