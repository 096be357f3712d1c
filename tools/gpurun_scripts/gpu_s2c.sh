set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/s2c_tdense.log 2>&1
tail -5 gpurun_out/s2c_tdense.log
timeout 600 python bench.py --config 3 --dense-k 5 --steps 1 --no-cpu-baseline > gpurun_out/s2c_c4_k5.log 2>&1
timeout 600 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2c_c4c64_k5_tc.log 2>&1
TCX_DENSE_TC=0 timeout 600 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2c_c4c64_k5_fma.log 2>&1
timeout 600 python bench.py --config 3 --dense-k 4 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2c_c4c64_k4.log 2>&1
timeout 600 python bench.py --config 1 --dense-k 4 --steps 3 --no-cpu-baseline > gpurun_out/s2c_c2_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dense_fwd_tc -s 20 -c 1 -o gpurun_out/prof_densetc_s2c -f python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc_s2c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dense_fwd_kernel -s 20 -c 1 -o gpurun_out/prof_densek2_s2c -f python bench.py --config 3 --dense-k 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k2_s2c.log 2>&1
for f in gpurun_out/s2c_c*.log; do echo $f; tail -1 $f | cut -c1-200; done
