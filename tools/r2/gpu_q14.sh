# cfg3 line-level attribution of the backward / forward pass 2 and cfg2 forward / backward pass 3
set -x
OUT=gpurun_out; mkdir -p $OUT/q14/d3 $OUT/q14/d2
N="ncu --set full --clock-control none --import-source on"
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
export TCX_JIT_CACHE=/tmp/q14_cache_$$
TCX_JIT_DUMP=$OUT/q14/d3 timeout 900 $N -k regex:'tcx_jit_bwd_2$' -s 3 -c 1 -o $OUT/q14/c3_bwd2 -f $BB --config 2 > $OUT/q14/n1.log 2>&1
TCX_JIT_DUMP=$OUT/q14/d3 timeout 900 $N -k regex:'tcx_jit_fwd_2$' -s 3 -c 1 -o $OUT/q14/c3_fwd2 -f $BB --config 2 > $OUT/q14/n2.log 2>&1
TCX_JIT_DUMP=$OUT/q14/d2 timeout 900 $N -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/q14/c2_fwd3 -f $BB --config 1 > $OUT/q14/n3.log 2>&1
for k in c3_bwd2:d3:bwd_2 c3_fwd2:d3:fwd_2 c2_fwd3:d2:fwd_3; do
  IFS=: read r d n <<< "$k"
  python tools/r2/ncu_lines.py $OUT/q14/$r.ncu-rep $OUT/q14/$d/tcx_jit_$n.cubin $OUT/q14/$d/tcx_jit_$n.cu 60 > $OUT/q14/lines_$r.txt 2>&1
done
rm -f $OUT/q14/*.ncu-rep $OUT/q14/d2/*.cubin
du -sh $OUT/q14
