set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t20.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b20_c2.log 2>&1
TCX_DIAG_NOLUT=1 timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b20_c2_nolut.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/b20_c3.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b20_c1.log 2>&1
tail -3 gpurun_out/t20.log
