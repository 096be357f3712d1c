# cfg3 ncu (regrouped + deferred factors) and cfg4 A/B (tan, regroup)
set -x
OUT=gpurun_out; mkdir -p $OUT/ncu3
B="python bench.py --no-cpu-baseline"
timeout 900 $B --config 3 --steps 2 > $OUT/q3_c4.log 2>&1
TCX_NO_TAN=1 timeout 900 $B --config 3 --steps 2 > $OUT/q3_c4_notan.log 2>&1
TCX_NO_DIAG_REGROUP=1 timeout 900 $B --config 3 --steps 2 > $OUT/q3_c4_noreg.log 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:'tcx_jit_bwd_3$' -s 3 -c 1 -o $OUT/ncu3/c3_bwd3 -f $B --config 2 --steps 1 --warmup 3 > $OUT/ncu3/n1.log 2>&1
timeout 900 $N -k regex:'tcx_jit_fwd_3$' -s 3 -c 1 -o $OUT/ncu3/c3_fwd3 -f $B --config 2 --steps 1 --warmup 3 > $OUT/ncu3/n2.log 2>&1
python tools/r2/ncu_summary.py $OUT/ncu_r2_q3.md "cfg3 after diagonal regroup + deferred factors: forward / backward pass 3" $OUT/ncu3/c3_fwd3.ncu-rep $OUT/ncu3/c3_bwd3.ncu-rep > $OUT/ncu3/sum.log 2>&1
for r in $OUT/ncu3/*.ncu-rep; do ncu -i $r --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
out=[]
for k,x in zip(h,v):
    if 'warps_issue_stalled' in k and 'per_issue_active' in k:
        try: out.append((float(x),k))
        except: pass
print('$r', [(k.split('stalled_')[1].split('_per')[0], round(x,2)) for x,k in sorted(out,reverse=True)[:8]])
" >> $OUT/ncu_r2_q3_stalls.txt; done
for f in $OUT/q3_c4*.log; do echo "== $f"; tail -1 $f | cut -c1-200; done
