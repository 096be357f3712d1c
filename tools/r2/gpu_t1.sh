# session-3 re-entry check: full GPU suite + cfg2/cfg3 lines on the restored tree
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/t1_c2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --config 2 --steps 3 > gpurun_out/t1_c3.log 2>&1
for f in gpurun_out/t1_c*.log; do echo "== $f"; tail -1 $f | cut -c1-160; done
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t1_tests.log 2>&1
tail -5 gpurun_out/t1_tests.log
