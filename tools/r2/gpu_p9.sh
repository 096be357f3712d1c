# cut tables for LUT ops: parity + cfg3 bench (with / without tables)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_noise.py -x -q -p no:cacheprovider -k "qaoa or cfg3 or random or fuzz or grad or table" > gpurun_out/p9_tests.log 2>&1
tail -5 gpurun_out/p9_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B --config 2 --steps 3 > gpurun_out/p9_c3.log 2>&1
TCX_NO_CUT_TABLE=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/p9_c3_nocut.log 2>&1
for f in gpurun_out/p9_c*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.4g ms %.4f' % (d['value'], d['ms_per_step']), {k:d['config']['plan'][k] for k in ('tile_bits','reg_bits','fwd_passes','stages')})
print(' roof', {k: (round(r.get(k),3) if isinstance(r.get(k),float) else r.get(k)) for k in ('bound','frac','achieved')}, (r.get('survey_model') or {}).get('frac'))
print(' kernels', {k:(round(v['ms'],4), round(v['tflops'],2), round(v['gbs'])) for k,v in d['kernels'].items()})" 2>&1 | tail -3; done
