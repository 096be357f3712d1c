set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s3b_t.log 2>&1
tail -3 gpurun_out/s3b_t.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/s3b_c2.log 2>&1
TCX_CX_BONUS=0 timeout 900 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/s3b_c2_nobonus.log 2>&1
timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s3b_c3.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/s3b_c4.log 2>&1
for f in gpurun_out/s3b_c*.log; do echo $f; tail -1 $f | cut -c1-120; done
