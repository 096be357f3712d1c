set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q > gpurun_out/s3d_t.log 2>&1
tail -30 gpurun_out/s3d_t.log
