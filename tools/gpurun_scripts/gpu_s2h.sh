set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q -k "k5 or tensor or state_random" > gpurun_out/s2h_tdense.log 2>&1
tail -5 gpurun_out/s2h_tdense.log
timeout 600 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2h_c4c64_k5_tc.log 2>&1
tail -1 gpurun_out/s2h_c4c64_k5_tc.log | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:dense_fwd_tc -s 20 -c 1 -o gpurun_out/prof_densetc_s2h -f python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc_s2h.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s2h_c3.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_s2h_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcx_jit_bwd -s 20 -c 1 -o gpurun_out/prof_c3bwd_s2h -f python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3_s2h.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcx_jit_fwd -s 20 -c 1 -o gpurun_out/prof_c3fwd_s2h -f python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3f_s2h.log 2>&1
ls gpurun_out
