# ncu evidence (round 2 code), summarised on the box (reports are large): cfg2 headline fwd/bwd
# (source level), cfg2 per-gate fwd/bwd (DRAM bytes vs algorithmic), cluster megakernels
set -x
OUT=gpurun_out; mkdir -p $OUT/ncu12
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/ncu12/c2_bwd3 -f $B --config 1 > $OUT/ncu12/n1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/ncu12/c2_fwd3 -f $B --config 1 > $OUT/ncu12/n2.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_bwd_200$' -s 3 -c 1 -o $OUT/ncu12/c2pg_bwd200 -f $B --config 1 --max-ops-per-pass 1 > $OUT/ncu12/n3.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_fwd_200$' -s 3 -c 1 -o $OUT/ncu12/c2pg_fwd200 -f $B --config 1 --max-ops-per-pass 1 > $OUT/ncu12/n4.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_cluster' -s 3 -c 1 -o $OUT/ncu12/cl14 -f $B --config 1 --qubits 14 --cluster-bits 1 > $OUT/ncu12/n5.log 2>&1
ncu --set full --clock-control none -k regex:'tcx_jit_cluster' -s 3 -c 1 -o $OUT/ncu12/cl17 -f $B --config 1 --qubits 17 --cluster-bits 4 > $OUT/ncu12/n6.log 2>&1
python tools/r2/ncu_summary.py $OUT/ncu_r2_p12.md "round 2 ncu captures (tools/r2/gpu_p12.sh): cfg2 headline forward / backward pass 3, cfg2 per-gate setting (--max-ops-per-pass 1) pass 200, cluster-resident megakernels n = 14 (2 CTAs / row) and n = 17 (16 CTAs / row)" $OUT/ncu12/c2_fwd3.ncu-rep $OUT/ncu12/c2_bwd3.ncu-rep $OUT/ncu12/c2pg_fwd200.ncu-rep $OUT/ncu12/c2pg_bwd200.ncu-rep $OUT/ncu12/cl14.ncu-rep $OUT/ncu12/cl17.ncu-rep > $OUT/ncu12/sum.log 2>&1
for r in $OUT/ncu12/*.ncu-rep; do ncu -i $r --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
out=[]
for k,x in zip(h,v):
    if 'warps_issue_stalled' in k and 'per_issue_active' in k:
        try: out.append((float(x),k))
        except: pass
print('$r', [(k.split('stalled_')[1].split('_per')[0], round(x,2)) for x,k in sorted(out,reverse=True)[:6]])
" >> $OUT/ncu_r2_p12_stalls.txt; done
rm -f $OUT/ncu12/cl17.ncu-rep $OUT/ncu12/cl14.ncu-rep $OUT/ncu12/c2pg_*.ncu-rep
du -sh $OUT
