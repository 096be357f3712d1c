set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config 2 --tile-bits 13 --coalesce-bits 3 --steps 3 --no-cpu-baseline > gpurun_out/s2t_c3_t13c3.log 2>&1
timeout 900 python bench.py --config 2 --tile-bits 13 --coalesce-bits 2 --steps 3 --no-cpu-baseline > gpurun_out/s2t_c3_t13c2.log 2>&1
for f in gpurun_out/s2t_*.log; do echo $f; tail -1 $f | cut -c1-150; done
