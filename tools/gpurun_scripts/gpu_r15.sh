set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t15.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline --tile-bits 13 > gpurun_out/b15_c1_t13.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b15_c1.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline --tile-bits 13 > gpurun_out/b15_c2_t13.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline --tile-bits 12 > gpurun_out/b15_c3_t12.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline --tile-bits 13 > gpurun_out/b15_c3_t13.log 2>&1
tail -3 gpurun_out/t15.log
