# full GPU suite + every config line after regroup + deferred factors
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q4_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/q4_tests.log 2>&1
tail -8 gpurun_out/q4_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B > gpurun_out/q4_c2.log 2>&1
timeout 300 $B --config 0 --steps 50 > gpurun_out/q4_c1.log 2>&1
timeout 600 $B --config 2 --steps 3 > gpurun_out/q4_c3.log 2>&1
timeout 900 $B --config 3 --steps 2 > gpurun_out/q4_c4.log 2>&1
timeout 900 $B --config 4 --steps 3 > gpurun_out/q4_c5.log 2>&1
timeout 600 $B --config 1 --max-ops-per-pass 1 --steps 2 > gpurun_out/q4_c2pg.log 2>&1
for f in gpurun_out/q4_c*.log; do echo "== $f"; tail -1 $f | cut -c1-200; done
