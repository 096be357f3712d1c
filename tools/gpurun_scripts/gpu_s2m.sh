set -x
mkdir -p gpurun_out
TCX_DENSE_TC_WS=2 timeout 900 python -m pytest tests/test_gpu_dense.py -x -q -k "k5 or tensor or state_random or expect" > gpurun_out/s2m_tdense.log 2>&1
tail -5 gpurun_out/s2m_tdense.log
TCX_DENSE_TC_WS=2 timeout 600 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/s2m_c4c64_k5_ws.log 2>&1
tail -1 gpurun_out/s2m_c4c64_k5_ws.log | cut -c1-200
TCX_DENSE_TC_WS=2 ncu --set full --clock-control none --import-source on -k regex:dense_fwd_tc -s 20 -c 1 -o gpurun_out/prof_densetcws_s2m -f python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tcws_s2m.log 2>&1
