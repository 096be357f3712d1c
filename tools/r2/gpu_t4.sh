# 32-byte runs (coalesce_bits 2: cfg2 7 -> 6 passes, cfg5 7 -> 4) with / without interleaved
# tiles; cfg3 line-level ncu of the slow scattered-window passes (fwd_5 / bwd_5)
set -x
mkdir -p gpurun_out/t4/d3
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t4cache
timeout 600 $B --steps 5 --coalesce-bits 2 > gpurun_out/t4/c2_cb2.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 600 $B --steps 5 --coalesce-bits 2 > gpurun_out/t4/c2_cb2_ilv.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 600 $B --steps 5 --coalesce-bits 2 > gpurun_out/t4/c2_cb2_ilv_half.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/t4/c5.log 2>&1
timeout 900 $B --config 4 --steps 3 --coalesce-bits 2 > gpurun_out/t4/c5_cb2.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 900 $B --config 4 --steps 3 --coalesce-bits 2 > gpurun_out/t4/c5_cb2_ilv.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 900 $B --config 4 --steps 3 > gpurun_out/t4/c5_ilv.log 2>&1
for f in gpurun_out/t4/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
N="ncu --set full --clock-control none --import-source on"
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
TCX_JIT_TILE_ORDER=1 TCX_JIT_DUMP=gpurun_out/t4/d3 timeout 900 $N -k regex:'tcx_jit_bwd_5$' -s 3 -c 1 -o gpurun_out/t4/c3_bwd5 -f $BB --config 2 > gpurun_out/t4/n1.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_DUMP=gpurun_out/t4/d3 timeout 900 $N -k regex:'tcx_jit_fwd_5$' -s 3 -c 1 -o gpurun_out/t4/c3_fwd5 -f $BB --config 2 > gpurun_out/t4/n2.log 2>&1
for k in c3_bwd5:bwd_5 c3_fwd5:fwd_5; do
  IFS=: read r n <<< "$k"
  python tools/r2/ncu_lines.py gpurun_out/t4/$r.ncu-rep gpurun_out/t4/d3/tcx_jit_$n.cubin gpurun_out/t4/d3/tcx_jit_$n.cu 60 > gpurun_out/t4/lines_$r.txt 2>&1
  python tools/r2/ncu_summary.py gpurun_out/t4/sum_$r.md $r gpurun_out/t4/$r.ncu-rep > /dev/null 2>&1
  python tools/r2/ncu_sass_hot.py gpurun_out/t4/$r.ncu-rep > gpurun_out/t4/hot_$r.txt 2>&1
done
rm -f gpurun_out/t4/*.ncu-rep gpurun_out/t4/d3/*.cubin
ls -la gpurun_out/t4
