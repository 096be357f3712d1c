# ncu evidence for the lambda units (cfg2, cfg5) and the cfg5 N=1 backward pass
set -x
OUT=gpurun_out; mkdir -p $OUT/t15
N="ncu --set full --clock-control none --import-source on"
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
timeout 900 $N -k regex:'tcx_jit_lam' -s 1 -c 1 -o $OUT/t15/c2_lam -f $BB > $OUT/t15/n1.log 2>&1
timeout 1200 $N -k regex:'tcx_jit_lam' -s 3 -c 1 -o $OUT/t15/c5_lam -f $BB --config 4 > $OUT/t15/n2.log 2>&1
timeout 1200 $N -k regex:'tcx_jit_bwd_1$' -s 3 -c 1 -o $OUT/t15/c5_bwd1 -f $BB --config 4 > $OUT/t15/n3.log 2>&1
python tools/r2/ncu_summary.py $OUT/t15/ncu_r2_s3_t15.md "session-3: lambda units (cfg2, cfg5) and the cfg5 N=1 backward pass 1" $OUT/t15/c2_lam.ncu-rep $OUT/t15/c5_lam.ncu-rep $OUT/t15/c5_bwd1.ncu-rep > $OUT/t15/sum.log 2>&1
rm -f $OUT/t15/*.ncu-rep
tail -3 $OUT/t15/n1.log $OUT/t15/n2.log $OUT/t15/n3.log
