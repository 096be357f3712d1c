# final-tree sanity: smoke, parity / edge / tan subset, default bench line
set -x
mkdir -p gpurun_out/t14
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t14/smoke.log 2>&1; tail -1 gpurun_out/t14/smoke.log
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_tan.py tests/test_gpu_cluster.py -q -p no:cacheprovider > gpurun_out/t14/tests.log 2>&1
tail -2 gpurun_out/t14/tests.log
timeout 900 python bench.py > gpurun_out/t14/c2_default.log 2>&1
tail -1 gpurun_out/t14/c2_default.log | cut -c1-200
