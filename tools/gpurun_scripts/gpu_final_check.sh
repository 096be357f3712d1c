set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fc_t.log 2>&1
tail -3 gpurun_out/fc_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fc_bench.log 2>&1
tail -1 gpurun_out/fc_bench.log | cut -c1-200
