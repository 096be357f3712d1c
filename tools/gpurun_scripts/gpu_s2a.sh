set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2a_t.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s2a_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2a_ref.log 2>&1
timeout 1200 bash tools/profile_round.sh s2a 3 > gpurun_out/s2a_prof.log 2>&1
tail -3 gpurun_out/s2a_t.log; tail -2 gpurun_out/s2a_bench.log | cut -c1-400
