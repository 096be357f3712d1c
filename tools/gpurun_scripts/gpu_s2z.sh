set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:dense_bwd_kernel -s 30 -c 1 -o gpurun_out/prof_densebwd_s2z -f python bench.py --config 1 --dense-k 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dbwd_s2z.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dense_fwd_kernel -s 30 -c 1 -o gpurun_out/prof_densefwd_s2z -f python bench.py --config 1 --dense-k 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dfwd_s2z.log 2>&1
ls gpurun_out | grep s2z
