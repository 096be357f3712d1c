#!/bin/bash
# Round profile (run under gpurun, 1 GPU): launch list, per-launch DRAM traffic of the pass
# kernels, and one `ncu --set full` capture of the largest backward pass kernel.
# usage: tools/profile_round.sh TAG BIG_BWD_PASS [bench args]
TAG=${1:-r1}; BIG=${2:-3}; shift 2
OUT=gpurun_out; mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu-baseline $*"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/launches_bench_$TAG.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:'tcx_jit|pass_kernel' --log-file $OUT/traffic_$TAG.csv $BENCH > $OUT/traffic_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tcx_jit_bwd_${BIG}\$" -s 3 -c 1 \
    -o $OUT/prof_bwd_$TAG -f $BENCH > $OUT/ncu_bwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tcx_jit_fwd_${BIG}\$" -s 3 -c 1 \
    -o $OUT/prof_fwd_$TAG -f $BENCH > $OUT/ncu_fwd_$TAG.log 2>&1
ls -la $OUT
