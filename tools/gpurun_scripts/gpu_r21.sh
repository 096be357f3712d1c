set -x
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b21_c1.log 2>&1
TCX_JIT_NOOPQ=1 timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b21_c1_noopq.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b21_c2.log 2>&1
