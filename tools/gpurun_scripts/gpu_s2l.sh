set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2l_t.log 2>&1
tail -3 gpurun_out/s2l_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2l_smoke.log 2>&1
bash tools/gpu_final_r1.sh
