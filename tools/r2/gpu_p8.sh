# cfg1 latency variants (register bits, cluster) + cfg2 line with the SURVEY 8(d) model
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
for rb in 1 2 3; do timeout 300 $B --config 0 --steps 50 --reg-bits $rb > gpurun_out/p8_c1_r$rb.log 2>&1; done
timeout 300 $B --config 0 --steps 50 --reg-bits 1 --cluster-bits 1 > gpurun_out/p8_c1_r1_cl1.log 2>&1
timeout 300 $B --config 0 --steps 50 --reg-bits 2 --cluster-bits 2 > gpurun_out/p8_c1_r2_cl2.log 2>&1
timeout 300 $B --config 0 --steps 50 --reg-bits 3 --cluster-bits 3 > gpurun_out/p8_c1_r3_cl3.log 2>&1
timeout 600 $B --config 1 --steps 5 > gpurun_out/p8_c2.log 2>&1
for f in gpurun_out/p8_*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.4g ms %.4f' % (d['value'], d['ms_per_step']), {k:d['config']['plan'][k] for k in ('tile_bits','reg_bits','fwd_passes','stages')})
print(' roof', {k: (round(r.get(k),3) if isinstance(r.get(k),float) else r.get(k)) for k in ('bound','frac','achieved')}, r.get('survey_model'))
print(' kernels', {k:(round(v['ms'],4), round(v['tflops'],2)) for k,v in d['kernels'].items()})" 2>&1 | tail -3; done
