# exchange/compute overlap: sharded parity + cfg5 virtual-rank lines with / without overlap
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_shard.py tests/test_gpu_large.py -x -q -p no:cacheprovider -k "shard or sharded" > gpurun_out/p11_tests.log 2>&1
tail -5 gpurun_out/p11_tests.log
B="python bench.py --config 4 --steps 3"
for G in 2 8; do
  timeout 600 $B --virtual-ranks $G > gpurun_out/p11_c5v$G.log 2>&1
  TCX_XCHG_NO_OVERLAP=1 timeout 600 $B --virtual-ranks $G > gpurun_out/p11_c5v${G}_noov.log 2>&1
done
for f in gpurun_out/p11_c5*.log; do echo "== $f"; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.4g ms %.1f xchg %.1f share %.3f' % (d['value'], d['ms_per_step'], d['exchange_ms_per_step'], d['exchange_share']), d['config']['plan'])
print(' kernels', {k:(round(v['ms'],1), round(v['gbs'])) for k,v in d['kernels'].items()})" 2>&1 | tail -2; done
