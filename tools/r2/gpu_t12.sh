# session-3 final (depth-2 forward ring on): smoke, full GPU suite, every config line (default bench = cfg2 with cpu_baseline),
# reference arm, launch list of the default bench
set -x
OUT=gpurun_out; mkdir -p $OUT/t12
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/t12/smoke.log 2>&1; tail -2 $OUT/t12/smoke.log
B="python bench.py"
timeout 900 $B > $OUT/t12/c2_default.log 2>&1
timeout 300 $B --no-cpu-baseline --config 0 --steps 50 > $OUT/t12/c1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 2 --steps 3 > $OUT/t12/c3.log 2>&1
timeout 900 $B --no-cpu-baseline --config 3 --steps 2 > $OUT/t12/c4.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --steps 3 > $OUT/t12/c5.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --virtual-ranks 8 --steps 3 > $OUT/t12/c5_v8.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --max-ops-per-pass 1 --steps 2 > $OUT/t12/c2_pergate.log 2>&1
timeout 600 $B --no-cpu-baseline --config 5 --steps 50 > $OUT/t12/t7.log 2>&1
timeout 900 $B --impl reference --steps 2 --warmup 1 > $OUT/t12/ref.log 2>&1
for f in $OUT/t12/c*.log $OUT/t12/t7.log $OUT/t12/ref.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/t12/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/t12/ncu_list.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t12/tests.log 2>&1
tail -3 $OUT/t12/tests.log
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:'tcx_jit_fwd_200$' -s 1 -c 1 -o $OUT/t12/pg_fwd200 -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 --config 1 --max-ops-per-pass 1 > $OUT/t12/n1.log 2>&1
timeout 900 $N -k regex:'tcx_jit_bwd_2$' -s 3 -c 1 -o $OUT/t12/c2_bwd2 -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 > $OUT/t12/n2.log 2>&1
python tools/r2/ncu_summary.py $OUT/t12/ncu_r2_s3_t12.md "session-3 final: cfg2 per-gate forward pass 200 (two-deep prefetch ring), cfg2 backward pass 2 (the largest)" $OUT/t12/pg_fwd200.ncu-rep $OUT/t12/c2_bwd2.ncu-rep > $OUT/t12/sum.log 2>&1
rm -f $OUT/t12/*.ncu-rep
