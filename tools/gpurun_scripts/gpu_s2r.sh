set -x
mkdir -p gpurun_out
for rb in 2 3; do
  timeout 600 python bench.py --config 0 --reg-bits $rb --steps 50 --no-cpu-baseline > gpurun_out/s2r_c1_r$rb.log 2>&1
done
timeout 600 python bench.py --config 0 --tile-bits 9 --steps 50 --no-cpu-baseline > gpurun_out/s2r_c1_t9.log 2>&1
timeout 600 python bench.py --config 0 --tile-bits 8 --steps 50 --no-cpu-baseline > gpurun_out/s2r_c1_t8.log 2>&1
for f in gpurun_out/s2r_*.log; do echo $f; tail -1 $f | cut -c1-120; done
