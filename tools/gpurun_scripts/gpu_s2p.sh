set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s2p_t.log 2>&1
tail -5 gpurun_out/s2p_t.log
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2p_c2.log 2>&1
TCX_NO_UFOLD=1 timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2p_c2_nofold.log 2>&1
timeout 900 python bench.py --config 0 --steps 20 --no-cpu-baseline > gpurun_out/s2p_c1.log 2>&1
timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s2p_c3.log 2>&1
for f in gpurun_out/s2p_c*.log; do echo $f; tail -1 $f | cut -c1-150; done
