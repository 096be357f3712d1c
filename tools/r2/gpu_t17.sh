# final tree: smoke, default bench, cfg5 line, large + parity + shard tests
set -x
mkdir -p gpurun_out/t17
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t17/smoke.log 2>&1; tail -1 gpurun_out/t17/smoke.log
timeout 900 python bench.py --no-cpu-baseline --config 4 --steps 3 > gpurun_out/t17/c5.log 2>&1
tail -1 gpurun_out/t17/c5.log | cut -c1-160
timeout 1800 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_shard.py tests/test_gpu_edges.py -q -p no:cacheprovider > gpurun_out/t17/tests.log 2>&1
tail -2 gpurun_out/t17/tests.log
timeout 900 python bench.py > gpurun_out/t17/c2_default.log 2>&1
tail -1 gpurun_out/t17/c2_default.log | cut -c1-160
