# ncu: cfg3 backward / forward and cfg2 backward (current code) with SASS-level stall hot spots
set -x
OUT=gpurun_out; mkdir -p $OUT/ncu7
B="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/ncu7/c3_bwd3 -f $B --config 2 > $OUT/ncu7/n1.log 2>&1
timeout 900 $N -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/ncu7/c3_fwd3 -f $B --config 2 > $OUT/ncu7/n2.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/ncu7/c2_bwd3 -f $B --config 1 > $OUT/ncu7/n3.log 2>&1
python tools/r2/ncu_summary.py $OUT/ncu_r2_q7.md "round 2 q7: cfg3 backward / forward pass 3, cfg2 backward pass 3 (regroup, deferred factors, forward pipeline)" $OUT/ncu7/c3_fwd3.ncu-rep $OUT/ncu7/c3_bwd3.ncu-rep $OUT/ncu7/c2_bwd3.ncu-rep > $OUT/ncu7/sum.log 2>&1
for r in c3_bwd3 c3_fwd3 c2_bwd3; do python tools/r2/ncu_sass_hot.py $OUT/ncu7/$r.ncu-rep 40 > $OUT/ncu7/hot_$r.txt 2>&1; done
rm -f $OUT/ncu7/c3_fwd3.ncu-rep
