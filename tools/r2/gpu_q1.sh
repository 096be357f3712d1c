# re-entry check: full GPU suite + smoke + headline/cfg1/cfg3 lines on the restored tree
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q1_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/q1_tests.log 2>&1
tail -15 gpurun_out/q1_tests.log
B="python bench.py --no-cpu-baseline"
timeout 600 $B > gpurun_out/q1_c2.log 2>&1
timeout 300 $B --config 0 --steps 50 > gpurun_out/q1_c1.log 2>&1
timeout 600 $B --config 2 --steps 3 > gpurun_out/q1_c3.log 2>&1
for f in gpurun_out/q1_c*.log; do echo "== $f"; tail -1 $f | cut -c1-600; done
