set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "l2_row" > gpurun_out/s3f_t.log 2>&1
tail -5 gpurun_out/s3f_t.log
timeout 900 python bench.py --config 1 --dense-k 2 --l2-rows -1 --steps 2 --no-cpu-baseline > gpurun_out/s3f_c2k2_l2.log 2>&1
timeout 900 python bench.py --config 1 --l2-rows -1 --steps 5 --no-cpu-baseline > gpurun_out/s3f_c2_l2.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 1 --l2-rows -1 --steps 1 --no-cpu-baseline > gpurun_out/s3f_c2k1_l2.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 1 --steps 1 --no-cpu-baseline > gpurun_out/s3f_c2k1.log 2>&1
for f in gpurun_out/s3f_c*.log; do echo $f; tail -1 $f | cut -c1-120; done
