# round-2 consolidated measurement: suite, smoke, every config line, reference arm, launch list,
# ncu captures of the dominant kernels (summaries written on the box; reports are large)
set -x
OUT=gpurun_out; mkdir -p $OUT/q12
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/q12/smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/q12/tests.log 2>&1
tail -3 $OUT/q12/tests.log
B="python bench.py"
timeout 900 $B > $OUT/q12/c2_default.log 2>&1
timeout 300 $B --no-cpu-baseline --config 0 --steps 50 > $OUT/q12/c1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 2 --steps 3 > $OUT/q12/c3.log 2>&1
timeout 900 $B --no-cpu-baseline --config 3 --steps 2 > $OUT/q12/c4.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --steps 3 > $OUT/q12/c5.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --virtual-ranks 8 --steps 3 > $OUT/q12/c5_v8.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --max-ops-per-pass 1 --steps 2 > $OUT/q12/c2_pergate.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --qubits 14 --cluster-bits 1 --steps 5 > $OUT/q12/n14_cl1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 5 --steps 50 > $OUT/q12/t7.log 2>&1
timeout 900 $B --impl reference --steps 2 --warmup 1 > $OUT/q12/ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/q12/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/q12/ncu_list.log 2>&1
N="ncu --set full --clock-control none --import-source on"
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
timeout 900 $N -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/q12/c2_fwd3 -f $BB --config 1 > $OUT/q12/n1.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/q12/c2_bwd3 -f $BB --config 1 > $OUT/q12/n2.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_2$' -s 3 -c 1 -o $OUT/q12/c3_bwd2 -f $BB --config 2 > $OUT/q12/n3.log 2>&1
timeout 900 $N -k regex:'tcx_jit_fwd_2$' -s 3 -c 1 -o $OUT/q12/c3_fwd2 -f $BB --config 2 > $OUT/q12/n4.log 2>&1
timeout 900 $N -k regex:'tcx_jit_fwd_40$' -s 1 -c 1 -o $OUT/q12/c4_fwd40 -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 --config 3 > $OUT/q12/n5.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_200$' -s 3 -c 1 -o $OUT/q12/pg_bwd200 -f $BB --config 1 --max-ops-per-pass 1 > $OUT/q12/n6.log 2>&1
timeout 900 $N -k regex:'tcx_jit_mega' -s 3 -c 1 -o $OUT/q12/c1_mega -f $BB --config 0 > $OUT/q12/n7.log 2>&1
python tools/r2/ncu_summary.py $OUT/ncu_r2_final.md "round 2 final ncu captures: cfg2 forward / backward pass 3, cfg3 backward / forward pass 2, cfg4 forward pass 40, cfg2 per-gate backward pass 200, cfg1 megakernel" $OUT/q12/c2_fwd3.ncu-rep $OUT/q12/c2_bwd3.ncu-rep $OUT/q12/c3_bwd2.ncu-rep $OUT/q12/c3_fwd2.ncu-rep $OUT/q12/c4_fwd40.ncu-rep $OUT/q12/pg_bwd200.ncu-rep $OUT/q12/c1_mega.ncu-rep > $OUT/q12/sum.log 2>&1
for r in c2_bwd3 c3_bwd2 c4_fwd40; do python tools/r2/ncu_sass_hot.py $OUT/q12/$r.ncu-rep 25 > $OUT/q12/hot_$r.txt 2>&1; done
rm -f $OUT/q12/*.ncu-rep
ls $OUT/q12
