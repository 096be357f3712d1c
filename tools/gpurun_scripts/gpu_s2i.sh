set -x
mkdir -p gpurun_out
for tc in 12:2 13:3 13:2; do
  t=${tc%:*}; c=${tc#*:}
  timeout 600 python bench.py --config 1 --tile-bits $t --coalesce-bits $c --steps 5 --no-cpu-baseline > gpurun_out/s2i_c2_t${t}c${c}.log 2>&1
done
timeout 600 python bench.py --config 2 --tile-bits 12 --coalesce-bits 2 --steps 3 --no-cpu-baseline > gpurun_out/s2i_c3_t12c2.log 2>&1
for f in gpurun_out/s2i_*.log; do echo $f; tail -1 $f | cut -c1-150; done
