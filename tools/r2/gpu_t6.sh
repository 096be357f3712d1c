# session-3 consolidated measurement with the new defaults (auto run width, interleaved tiles,
# half pipeline): smoke, GPU suite, every config line, reference arm, launch list, ncu captures
set -x
OUT=gpurun_out; mkdir -p $OUT/t6
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/t6/smoke.log 2>&1; tail -2 $OUT/t6/smoke.log
B="python bench.py"
timeout 900 $B > $OUT/t6/c2_default.log 2>&1
timeout 600 $B --no-cpu-baseline --coalesce-bits 2 --steps 5 > $OUT/t6/c2_cb2.log 2>&1
timeout 300 $B --no-cpu-baseline --config 0 --steps 50 > $OUT/t6/c1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 2 --steps 3 > $OUT/t6/c3.log 2>&1
timeout 900 $B --no-cpu-baseline --config 3 --steps 2 > $OUT/t6/c4.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --steps 3 > $OUT/t6/c5.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --virtual-ranks 8 --steps 3 > $OUT/t6/c5_v8.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --max-ops-per-pass 1 --steps 2 > $OUT/t6/c2_pergate.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --qubits 14 --cluster-bits 1 --steps 5 > $OUT/t6/n14_cl1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 5 --steps 50 > $OUT/t6/t7.log 2>&1
for f in $OUT/t6/c*.log $OUT/t6/n14*.log $OUT/t6/t7.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/t6/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/t6/ncu_list.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file $OUT/t6/m_c3.csv $BB --config 2 > $OUT/t6/n0.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file $OUT/t6/m_c2.csv $BB --config 1 > $OUT/t6/n00.log 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/t6/c2_bwd3 -f $BB --config 1 > $OUT/t6/n2.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_2$' -s 3 -c 1 -o $OUT/t6/c3_bwd2 -f $BB --config 2 > $OUT/t6/n3.log 2>&1
timeout 900 $N -k regex:'tcx_jit_fwd_2$' -s 3 -c 1 -o $OUT/t6/c3_fwd2 -f $BB --config 2 > $OUT/t6/n4.log 2>&1
python tools/r2/ncu_summary.py $OUT/t6/ncu_r2_s3.md "session-3 ncu captures (auto run width, interleaved tiles, half pipeline): cfg2 backward pass 3, cfg3 backward / forward pass 2" $OUT/t6/c2_bwd3.ncu-rep $OUT/t6/c3_bwd2.ncu-rep $OUT/t6/c3_fwd2.ncu-rep > $OUT/t6/sum.log 2>&1
for r in c2_bwd3 c3_bwd2; do python tools/r2/ncu_sass_hot.py $OUT/t6/$r.ncu-rep 25 > $OUT/t6/hot_$r.txt 2>&1; done
rm -f $OUT/t6/*.ncu-rep
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t6/tests.log 2>&1
tail -3 $OUT/t6/tests.log
