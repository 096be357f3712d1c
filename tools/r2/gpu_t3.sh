# interleaved tile order (TCX_JIT_TILE_ORDER=1) x 128-byte runs x half pipeline on cfg3 / cfg2:
# parity subset (incl. chunked sharded exchanges) + A/B lines + per-kernel DRAM bytes
set -x
mkdir -p gpurun_out/t3
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t3cache
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_shard.py tests/test_gpu_terms.py tests/test_gpu_inputs.py -q -x -p no:cacheprovider > gpurun_out/t3/tests.log 2>&1
tail -3 gpurun_out/t3/tests.log
timeout 600 $B --config 2 --steps 3 > gpurun_out/t3/c3.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t3/c3_ilv.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 600 $B --config 2 --steps 3 --coalesce-bits 4 > gpurun_out/t3/c3_ilv_cb4.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 600 $B --config 2 --steps 3 > gpurun_out/t3/c3_ilv_half.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 600 $B --config 2 --steps 3 --coalesce-bits 4 > gpurun_out/t3/c3_ilv_half_cb4.log 2>&1
timeout 600 $B --steps 5 > gpurun_out/t3/c2.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 600 $B --steps 5 > gpurun_out/t3/c2_ilv.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 600 $B --steps 5 > gpurun_out/t3/c2_ilv_half.log 2>&1
TCX_JIT_TILE_ORDER=1 TCX_JIT_HALFPIPE=1 timeout 600 $B --steps 5 --coalesce-bits 4 > gpurun_out/t3/c2_ilv_half_cb4.log 2>&1
for f in gpurun_out/t3/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum
BB="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
TCX_JIT_TILE_ORDER=1 timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t3/m_c3_ilv.csv $BB --config 2 > gpurun_out/t3/n1.log 2>&1
TCX_JIT_TILE_ORDER=1 timeout 900 ncu --metrics $M --clock-control none -k regex:tcx_jit -s 0 -c 16 --csv --log-file gpurun_out/t3/m_c2_ilv.csv $BB --config 1 > gpurun_out/t3/n2.log 2>&1
ls -la gpurun_out/t3
