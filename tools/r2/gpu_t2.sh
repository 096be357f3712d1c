# half pipeline for two-state passes (TCX_JIT_HALFPIPE), psi/lambda placement (TCX_LAM_PAD),
# L2 prefetch and 128-byte runs on cfg3 / cfg2: parity subset + A/B lines + per-kernel DRAM bytes
set -x
mkdir -p gpurun_out/t2
B="python bench.py --no-cpu-baseline"
PAD=1049856
TCX_JIT_HALFPIPE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py -q -x -p no:cacheprovider > gpurun_out/t2/tests_half.log 2>&1
tail -3 gpurun_out/t2/tests_half.log
timeout 600 $B --config 2 --steps 3 > gpurun_out/t2/c3.log 2>&1
TCX_JIT_HALFPIPE=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t2/c3_half.log 2>&1
TCX_LAM_PAD=$PAD timeout 600 $B --config 2 --steps 3 > gpurun_out/t2/c3_pad.log 2>&1
TCX_JIT_PREFETCH=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t2/c3_pf.log 2>&1
timeout 600 $B --config 2 --steps 3 --coalesce-bits 4 > gpurun_out/t2/c3_cb4.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t2/c2.log 2>&1
TCX_JIT_HALFPIPE=1 timeout 600 $B --steps 5 > gpurun_out/t2/c2_half.log 2>&1
TCX_LAM_PAD=$PAD timeout 600 $B --steps 5 > gpurun_out/t2/c2_pad.log 2>&1
for f in gpurun_out/t2/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t2/m_c3.csv $BB --config 2 > gpurun_out/t2/n1.log 2>&1
TCX_LAM_PAD=$PAD timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t2/m_c3_pad.csv $BB --config 2 > gpurun_out/t2/n2.log 2>&1
TCX_JIT_HALFPIPE=1 timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t2/m_c3_half.csv $BB --config 2 > gpurun_out/t2/n4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t2/m_c2.csv $BB --config 1 > gpurun_out/t2/n3.log 2>&1
ls -la gpurun_out/t2
