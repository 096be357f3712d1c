set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t16.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b16_c1.log 2>&1
TCX_JIT_NOPREFETCH=1 timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b16_c1_nopf.log 2>&1
TCX_JIT_NSUB=2 timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b16_c1_nsub2.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b16_c2.log 2>&1
timeout 600 python bench.py --config 0 --steps 50 --no-cpu-baseline > gpurun_out/b16_c0.log 2>&1
tail -3 gpurun_out/t16.log
