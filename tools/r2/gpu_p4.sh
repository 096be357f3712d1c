# ncu evidence: cfg3 fwd/bwd passes (source level), cfg1 megakernel, cfg2 lambda kernel, exchange swap
set -x
OUT=gpurun_out; mkdir -p $OUT
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/p4_c3_bwd3 -f $B --config 2 > $OUT/p4_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/p4_c3_fwd3 -f $B --config 2 > $OUT/p4_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_mega' -s 3 -c 1 -o $OUT/p4_c3_fusedlast -f $B --config 2 > $OUT/p4_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_mega' -s 5 -c 1 -o $OUT/p4_c1_mega -f $B --config 0 --graph 0 > $OUT/p4_ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_lam' -s 3 -c 1 -o $OUT/p4_c2_lam -f $B --config 1 > $OUT/p4_ncu5.log 2>&1
ncu --set full --clock-control none -k regex:'virtual_swap' -s 2 -c 1 -o $OUT/p4_c5_swap -f python bench.py --config 4 --virtual-ranks 2 --batch-qubits 27 --steps 1 --warmup 3 > $OUT/p4_ncu6.log 2>&1
ls -la $OUT/p4_*
