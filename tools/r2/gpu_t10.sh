# cfg3 as the p + 1 = 6-pass plan (8192-amplitude tiles, 32-byte runs, every window a TMA box)
# with the half pipeline now allowed for one-CTA-per-SM kernels
set -x
mkdir -p gpurun_out/t10
B="python bench.py --no-cpu-baseline"
export TCX_JIT_CACHE=/tmp/t10cache
timeout 600 $B --config 2 --steps 3 > gpurun_out/t10/c3.log 2>&1
timeout 600 $B --config 2 --steps 3 --tile-bits 13 --coalesce-bits 2 > gpurun_out/t10/c3_t13.log 2>&1
TCX_JIT_HALFPIPE=0 timeout 600 $B --config 2 --steps 3 --tile-bits 13 --coalesce-bits 2 > gpurun_out/t10/c3_t13_nohalf.log 2>&1
timeout 600 $B --config 2 --steps 3 --tile-bits 13 --coalesce-bits 3 > gpurun_out/t10/c3_t13_cb3.log 2>&1
timeout 600 $B --steps 5 --tile-bits 13 > gpurun_out/t10/c2_t13.log 2>&1
for f in gpurun_out/t10/c*.log; do echo "== $f"; tail -1 $f | cut -c1-140; done
