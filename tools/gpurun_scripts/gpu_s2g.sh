set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2g_t.log 2>&1
tail -3 gpurun_out/s2g_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2g_smoke.log 2>&1
timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s2g_c3.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/s2g_c4.log 2>&1
timeout 900 python bench.py --config 0 --steps 10 > gpurun_out/s2g_c1.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 2 --steps 2 --no-cpu-baseline > gpurun_out/s2g_c2_k2.log 2>&1
timeout 900 python bench.py > gpurun_out/s2g_bench.log 2>&1
timeout 1200 bash tools/profile_round.sh s2g 3 > gpurun_out/s2g_prof.log 2>&1
for f in gpurun_out/s2g_c*.log gpurun_out/s2g_bench.log; do echo $f; tail -1 $f | cut -c1-250; done
