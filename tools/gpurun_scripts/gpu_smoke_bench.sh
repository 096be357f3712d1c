set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sb_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/sb_bench.log 2>&1
tail -1 gpurun_out/sb_smoke.log; tail -1 gpurun_out/sb_bench.log | cut -c1-150
