set -x
mkdir -p gpurun_out
for v in 4 16 32 64; do
  TCX_TPC=$v timeout 900 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s3e_c2_tpc$v.log 2>&1
done
for v in 16 64; do
  TCX_TPC=$v timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s3e_c3_tpc$v.log 2>&1
done
for f in gpurun_out/s3e_*.log; do echo $f; tail -1 $f | cut -c1-100; done
