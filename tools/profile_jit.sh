#!/bin/bash
# ncu captures of the JIT pass kernels (run under gpurun).  usage: tools/profile_jit.sh TAG PASS [bench args]
TAG=${1:-r1}; PASS=${2:-3}; shift 2
OUT=gpurun_out; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > $OUT/launches_bench_$TAG.log 2>&1
for K in bwd fwd; do
ncu --set full --clock-control none --import-source on -k regex:"tcx_jit_${K}_${PASS}\$" -s 3 -c 1 \
    -o $OUT/prof_${K}_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_${K}_$TAG.log 2>&1
done
ls -la $OUT
