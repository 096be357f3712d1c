# cluster-resident states: parity + benches
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_cluster.py -x -q -p no:cacheprovider > gpurun_out/p5_tests.log 2>&1
tail -15 gpurun_out/p5_tests.log
B="python bench.py --no-cpu-baseline"
timeout 300 $B --config 0 --steps 50 > gpurun_out/p5_c1_base.log 2>&1
timeout 300 $B --config 0 --steps 50 --cluster-bits 1 > gpurun_out/p5_c1_cb1.log 2>&1
timeout 300 $B --config 0 --steps 50 --cluster-bits 2 > gpurun_out/p5_c1_cb2.log 2>&1
for q in 14 16 17; do
  cb=$((q-13))
  timeout 600 $B --config 1 --qubits $q --steps 5 > gpurun_out/p5_n${q}_win.log 2>&1
  timeout 600 $B --config 1 --qubits $q --steps 5 --l2-rows -1 > gpurun_out/p5_n${q}_l2.log 2>&1
  timeout 900 $B --config 1 --qubits $q --steps 5 --cluster-bits $cb > gpurun_out/p5_n${q}_cl.log 2>&1
done
for f in gpurun_out/p5_c1*.log gpurun_out/p5_n*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.1f ms %.3f' % (d['value'], d['ms_per_step']), {k:d['config']['plan'][k] for k in ('tile_bits','fwd_passes')})
print(' roof', {k: (round(r.get(k),3) if isinstance(r.get(k),float) else r.get(k)) for k in ('bound','frac','achieved','hbm_achieved_gbs')})
print(' kernels', {k:(round(v['ms'],3), round(v['gbs']), round(v['tflops'],1)) for k,v in d['kernels'].items()})" 2>&1 | tail -3; done
