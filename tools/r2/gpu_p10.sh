# ncu evidence (round 2 code): cfg2 headline fwd/bwd (source level), cfg2 per-gate bwd (DRAM bytes
# vs algorithmic), cluster megakernels n=14 / n=17, cfg5 n=33 backward pass
set -x
OUT=gpurun_out; mkdir -p $OUT
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/p10_c2_bwd3 -f $B --config 1 > $OUT/p10_n1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/p10_c2_fwd3 -f $B --config 1 > $OUT/p10_n2.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_bwd_200$' -s 3 -c 1 -o $OUT/p10_c2pg_bwd -f $B --config 1 --max-ops-per-pass 1 > $OUT/p10_n3.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_fwd_200$' -s 3 -c 1 -o $OUT/p10_c2pg_fwd -f $B --config 1 --max-ops-per-pass 1 > $OUT/p10_n3b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_cluster' -s 3 -c 1 -o $OUT/p10_cl14 -f $B --config 1 --qubits 14 --cluster-bits 1 > $OUT/p10_n4.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_cluster' -s 3 -c 1 -o $OUT/p10_cl17 -f $B --config 1 --qubits 17 --cluster-bits 4 > $OUT/p10_n5.log 2>&1
ls -la $OUT/p10_*
