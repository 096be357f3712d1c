# full GPU suite after stage lookahead + opt-in multi-box (module-load failure check) + cfg3 line
set -x
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/q18_tests.log 2>&1
tail -5 gpurun_out/q18_tests.log
timeout 600 python bench.py --no-cpu-baseline --config 2 --steps 3 > gpurun_out/q18_c3.log 2>&1
tail -1 gpurun_out/q18_c3.log | cut -c1-150
