#!/bin/bash
# Run on the GPU box (gpurun): launch list + one full ncu capture of the top kernels.
# usage: tools/profile_ncu.sh TAG BWD_SKIP FWD_SKIP [bench args...]
set -x
TAG=${1:-r1}; BS=${2:-28}; FS=${3:-30}; shift 3
OUT=gpurun_out
mkdir -p $OUT
: ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $OUT/launches_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'pass_kernel<float, .int.4, .int.1>' -s $BS -c 1 \
    -o $OUT/prof_bwd_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_bwd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'pass_kernel<float, .int.4, .int.0>' -s $FS -c 1 \
    -o $OUT/prof_fwd_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_fwd_$TAG.log 2>&1
ls -la $OUT
