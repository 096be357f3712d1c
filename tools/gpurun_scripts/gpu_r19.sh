set -x
TCX_JIT_MINB=2 timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline --reg-bits 3 > gpurun_out/b19_c1_r3m2.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline --reg-bits 3 > gpurun_out/b19_c1_r3m1.log 2>&1
timeout 900 python tools/ab_parts.py 2 > gpurun_out/ab19_c2.log 2>&1
