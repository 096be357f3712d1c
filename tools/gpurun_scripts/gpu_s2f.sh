set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/s2f_tdense.log 2>&1
tail -5 gpurun_out/s2f_tdense.log
timeout 600 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2f_c4c64_k5_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dense_fwd_tc -s 20 -c 1 -o gpurun_out/prof_densetc_s2f -f python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc_s2f.log 2>&1
tail -1 gpurun_out/s2f_c4c64_k5_tc.log | cut -c1-200
