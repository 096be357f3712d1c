set -x
mkdir -p gpurun_out
timeout 600 python bench.py --config 0 --steps 50 --no-cpu-baseline > gpurun_out/s2q_c1_graph.log 2>&1
timeout 600 python bench.py --config 0 --steps 50 --graph 0 --no-cpu-baseline > gpurun_out/s2q_c1_eager.log 2>&1
TCX_NO_UFOLD=1 timeout 600 python bench.py --config 0 --steps 50 --no-cpu-baseline > gpurun_out/s2q_c1_nofold.log 2>&1
timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s2q_c2_graph.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 2 --steps 1 --no-cpu-baseline > gpurun_out/s2q_c2k2_graph.log 2>&1
timeout 600 python bench.py --config 2 --steps 2 --mode expect --no-cpu-baseline > gpurun_out/s2q_c3_expect.log 2>&1
for f in gpurun_out/s2q_*.log; do echo $f; tail -1 $f | cut -c1-150; done
