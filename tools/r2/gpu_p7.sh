# full GPU suite + one bench line per config after the lambda fix
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p7_tests.log 2>&1
tail -15 gpurun_out/p7_tests.log
B="python bench.py --no-cpu-baseline"
timeout 300 $B --config 0 --steps 50 > gpurun_out/p7_c1.log 2>&1
timeout 300 $B --config 0 --steps 50 --cluster-bits 2 > gpurun_out/p7_c1_cl2.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/p7_c4.log 2>&1
timeout 600 $B --config 4 --steps 3 > gpurun_out/p7_c5.log 2>&1
timeout 600 $B --config 1 --qubits 14 --steps 5 --cluster-bits 1 > gpurun_out/p7_n14_cl1.log 2>&1
timeout 600 $B --config 1 --qubits 17 --steps 5 --cluster-bits 4 > gpurun_out/p7_n17_cl4.log 2>&1
for f in gpurun_out/p7_c*.log gpurun_out/p7_n*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.3f ms %.4f' % (d['value'], d['ms_per_step']), {k:d['config']['plan'][k] for k in ('tile_bits','fwd_passes')}, d['config'].get('launch'))
print(' roof', {k: (round(r.get(k),3) if isinstance(r.get(k),float) else r.get(k)) for k in ('bound','frac','achieved','hbm_achieved_gbs','kernel')})
print(' kernels', {k:(round(v['ms'],3), round(v['gbs']), round(v['tflops'],1)) for k,v in d['kernels'].items()})" 2>&1 | tail -3; done
