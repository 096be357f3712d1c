set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/s2b_tdense.log 2>&1
tail -5 gpurun_out/s2b_tdense.log
for k in 5 4 3 2; do
  timeout 600 python bench.py --config 3 --dense-k $k --steps 1 --no-cpu-baseline > gpurun_out/s2b_c4_k$k.log 2>&1
done
timeout 600 python bench.py --config 1 --dense-k 4 --steps 3 --no-cpu-baseline > gpurun_out/s2b_c2_k4.log 2>&1
timeout 600 python bench.py --config 1 --dense-k 2 --steps 3 --no-cpu-baseline > gpurun_out/s2b_c2_k2.log 2>&1
timeout 900 python bench.py --config 3 --dense-k 1 --steps 1 --no-cpu-baseline > gpurun_out/s2b_c4_k1.log 2>&1
for f in gpurun_out/s2b_c*.log; do echo $f; tail -1 $f | cut -c1-300; done
