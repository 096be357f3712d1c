set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s3h_t.log 2>&1
tail -3 gpurun_out/s3h_t.log
timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s3h_c3.log 2>&1
TCX_NO_FUSE_LAST=1 timeout 900 python bench.py --config 2 --steps 3 --no-cpu-baseline > gpurun_out/s3h_c3_nofuse.log 2>&1
for f in gpurun_out/s3h_c*.log; do echo $f; tail -1 $f | cut -c1-120; done
