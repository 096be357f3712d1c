set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t18.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b18_c2.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/b18_c3.log 2>&1
timeout 900 bash tools/profile_jit.sh r2 3 --config 1
tail -3 gpurun_out/t18.log
