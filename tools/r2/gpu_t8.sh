# session-3 final: smoke, full GPU suite, every config line (default bench = cfg2 with cpu_baseline),
# reference arm, launch list of the default bench
set -x
OUT=gpurun_out; mkdir -p $OUT/t8
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/t8/smoke.log 2>&1; tail -2 $OUT/t8/smoke.log
B="python bench.py"
timeout 900 $B > $OUT/t8/c2_default.log 2>&1
timeout 300 $B --no-cpu-baseline --config 0 --steps 50 > $OUT/t8/c1.log 2>&1
timeout 600 $B --no-cpu-baseline --config 2 --steps 3 > $OUT/t8/c3.log 2>&1
timeout 900 $B --no-cpu-baseline --config 3 --steps 2 > $OUT/t8/c4.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --steps 3 > $OUT/t8/c5.log 2>&1
timeout 900 $B --no-cpu-baseline --config 4 --virtual-ranks 8 --steps 3 > $OUT/t8/c5_v8.log 2>&1
timeout 600 $B --no-cpu-baseline --config 1 --max-ops-per-pass 1 --steps 2 > $OUT/t8/c2_pergate.log 2>&1
timeout 600 $B --no-cpu-baseline --config 5 --steps 50 > $OUT/t8/t7.log 2>&1
timeout 900 $B --impl reference --steps 2 --warmup 1 > $OUT/t8/ref.log 2>&1
for f in $OUT/t8/c*.log $OUT/t8/t7.log $OUT/t8/ref.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/t8/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/t8/ncu_list.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t8/tests.log 2>&1
tail -3 $OUT/t8/tests.log
