set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_shard.py tests/test_gpu_large.py -x -q -m gpu -p no:cacheprovider > gpurun_out/p2_tests.log 2>&1
tail -15 gpurun_out/p2_tests.log
timeout 600 python bench.py --config 4 --steps 3 > gpurun_out/p2_c5n1.log 2>&1
timeout 600 python bench.py --config 4 --virtual-ranks 2 --steps 3 > gpurun_out/p2_c5v2.log 2>&1
timeout 600 python bench.py --config 4 --virtual-ranks 8 --steps 3 > gpurun_out/p2_c5v8.log 2>&1
for f in gpurun_out/p2_c5*.log; do echo $f; tail -2 $f | cut -c1-1500; done
