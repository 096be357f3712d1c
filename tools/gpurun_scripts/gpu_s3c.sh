set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config 2 --reg-bits 3 --steps 3 --no-cpu-baseline > gpurun_out/s3c_c3_r3.log 2>&1
timeout 900 python bench.py --config 1 --reg-bits 3 --steps 3 --no-cpu-baseline > gpurun_out/s3c_c2_r3.log 2>&1
TCX_JIT_MINB=1 timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s3c_c3_minb1.log 2>&1
for f in gpurun_out/s3c_*.log; do echo $f; tail -1 $f | cut -c1-120; done
