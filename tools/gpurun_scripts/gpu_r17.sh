set -x
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b17_c1.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline --coalesce-bits 2 > gpurun_out/b17_c1_cb2.log 2>&1
TCX_JIT_NSUB=2 timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b17_c1_nsub2.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline --coalesce-bits 2 > gpurun_out/b17_c2_cb2.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline --coalesce-bits 1 > gpurun_out/b17_c2_cb1.log 2>&1
