# full GPU suite + benches after: specialised fused lambda, one-slot LUT backward, auto pipe,
# cluster 2-CTA/SM variant
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p6_tests.log 2>&1
tail -15 gpurun_out/p6_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --config 2 --steps 3 > gpurun_out/p6_c3.log 2>&1
timeout 600 $B --config 1 --steps 5 > gpurun_out/p6_c2.log 2>&1
timeout 900 $B --config 1 --steps 2 --max-ops-per-pass 1 > gpurun_out/p6_c2_unfused.log 2>&1
timeout 900 $B --config 1 --steps 2 --max-ops-per-pass 1 --graph 0 > gpurun_out/p6_c2_unfused_eager.log 2>&1
timeout 600 $B --config 1 --qubits 16 --steps 5 --cluster-bits 4 > gpurun_out/p6_n16_cl4.log 2>&1
timeout 600 $B --config 1 --qubits 15 --steps 5 --cluster-bits 3 > gpurun_out/p6_n15_cl3.log 2>&1
timeout 600 $B --config 1 --qubits 15 --steps 5 > gpurun_out/p6_n15_win.log 2>&1
for f in gpurun_out/p6_c*.log gpurun_out/p6_n*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.1f ms %.4f' % (d['value'], d['ms_per_step']), {k:d['config']['plan'][k] for k in ('tile_bits','fwd_passes')}, d['config'].get('launch'))
print(' roof', {k: (round(r.get(k),3) if isinstance(r.get(k),float) else r.get(k)) for k in ('bound','frac','achieved','hbm_achieved_gbs','kernel')})
print(' kernels', {k:(round(v['ms'],3), round(v['gbs']), round(v['tflops'],1)) for k,v in d['kernels'].items()})" 2>&1 | tail -3; done
