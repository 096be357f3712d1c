set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config 1 --dense-k 2 --l2-rows -1 --graph 1 --steps 2 --no-cpu-baseline > gpurun_out/s3g_c2k2_l2_graph.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 2 --graph 1 --steps 2 --no-cpu-baseline > gpurun_out/s3g_c2k2_graph.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 4 --l2-rows -1 --graph 1 --steps 2 --no-cpu-baseline > gpurun_out/s3g_c2k4_l2_graph.log 2>&1
for f in gpurun_out/s3g_c*.log; do echo $f; tail -1 $f | cut -c1-120; done
