# grouped tile order for huge rows (TCX_TILE_ORDER=g: blocked over groups of g CTAs, interleaved
# within a group) on cfg5's 32-byte-run plan; parity subset under the forced order
set -x
mkdir -p gpurun_out/t16
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t16cache
timeout 900 $B --config 4 --steps 3 > gpurun_out/t16/c5.log 2>&1
TCX_TILE_ORDER=4 timeout 900 $B --config 4 --steps 3 > gpurun_out/t16/c5_g4.log 2>&1
TCX_TILE_ORDER=2 timeout 900 $B --config 4 --steps 3 > gpurun_out/t16/c5_g2.log 2>&1
for f in gpurun_out/t16/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
TCX_TILE_ORDER=4 timeout 900 ncu --metrics $M --clock-control none -k regex:'tcx_jit_bwd_1$' -s 0 -c 1 --csv --log-file gpurun_out/t16/m_c5_g4.csv $B --steps 1 --warmup 3 --config 4 > gpurun_out/t16/n1.log 2>&1
TCX_TILE_ORDER=4 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -p no:cacheprovider -k "not cfg4" > gpurun_out/t16/tests.log 2>&1
tail -2 gpurun_out/t16/tests.log
