set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t14.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b14_c2.log 2>&1
TCX_U1_STRUCT=0 timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b14_c2_nostruct.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/b14_c1.log 2>&1
timeout 600 python bench.py --config 4 --virtual-ranks 2 --batch-qubits 28 --steps 3 > gpurun_out/b14_c4v.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/b14_c3jit.log 2>&1
tail -3 gpurun_out/t14.log
