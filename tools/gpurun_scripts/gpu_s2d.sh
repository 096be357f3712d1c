set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_inputs.py -x -q > gpurun_out/s2d_tin.log 2>&1
tail -3 gpurun_out/s2d_tin.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2d_t.log 2>&1
tail -3 gpurun_out/s2d_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2d_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s2d_bench.log 2>&1
tail -1 gpurun_out/s2d_bench.log | cut -c1-300
