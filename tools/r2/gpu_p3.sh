# pipelined TMA passes (TCX_JIT_PIPE) correctness + cfg3 / cfg2 variants
set -x
mkdir -p gpurun_out
TCX_JIT_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "multi_pass or qaoa or cfg3 or hea_heisenberg or structured or deterministic" > gpurun_out/p3_pipe_tests.log 2>&1
tail -3 gpurun_out/p3_pipe_tests.log
B="python bench.py --steps 3 --no-cpu-baseline"
timeout 600 $B --config 2 > gpurun_out/p3_c3_base.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 2 > gpurun_out/p3_c3_pipe.log 2>&1
timeout 600 $B --config 2 --tile-bits 13 --coalesce-bits 2 > gpurun_out/p3_c3_t13.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 2 --tile-bits 13 --coalesce-bits 2 > gpurun_out/p3_c3_t13_pipe.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 2 --tile-bits 12 --coalesce-bits 2 > gpurun_out/p3_c3_t12c2_pipe.log 2>&1
timeout 600 $B --config 1 --max-ops-per-pass 20 > gpurun_out/p3_c2_pl.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 1 --max-ops-per-pass 20 > gpurun_out/p3_c2_pl_pipe.log 2>&1
timeout 600 $B --config 1 > gpurun_out/p3_c2_base.log 2>&1
TCX_JIT_PIPE=1 timeout 600 $B --config 1 > gpurun_out/p3_c2_pipe.log 2>&1
for f in gpurun_out/p3_c*.log; do echo $f; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('value %.1f ms %.1f plan %s' % (d['value'], d['ms_per_step'], d['config']['plan']))
print(' roof', {k: r.get(k) for k in ('bound','achieved','frac','kernel','hbm_achieved_gbs')})
print(' kernels', {k:(round(v['ms'],1), round(v['gbs']), round(v['tflops'],1)) for k,v in d['kernels'].items()})" 2>&1 | tail -4; done
