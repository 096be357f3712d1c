set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s2j_t.log 2>&1
tail -3 gpurun_out/s2j_t.log
timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s2j_c3.log 2>&1
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2j_c2.log 2>&1
for f in gpurun_out/s2j_c*.log; do echo $f; tail -1 $f | cut -c1-150; done
