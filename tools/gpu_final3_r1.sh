# Round-1 final measurement set v2 (one GPU): full GPU suite + smoke, bench lines for every
# config (CUDA-graph replay), the reference arm, and the ncu launch list / traffic / full
# captures of the headline bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin3_smi.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin3_t.log 2>&1
tail -3 gpurun_out/fin3_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin3_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin3_ref.log 2>&1
timeout 600 python bench.py --config 0 --steps 50 > gpurun_out/fin3_c1.log 2>&1
timeout 900 python bench.py --config 2 --steps 3 > gpurun_out/fin3_c3.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/fin3_c4.log 2>&1
timeout 900 python bench.py --config 3 --dense-k 2 --steps 1 --no-cpu-baseline > gpurun_out/fin3_c4_k2.log 2>&1
timeout 900 python bench.py --config 3 --dense-k 5 --dtype c64 --steps 1 --no-cpu-baseline > gpurun_out/fin3_c4c64_k5.log 2>&1
timeout 900 python bench.py --config 4 --virtual-ranks 2 --steps 3 > gpurun_out/fin3_c5v2.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 2 --steps 2 --no-cpu-baseline > gpurun_out/fin3_c2_k2.log 2>&1
timeout 600 python bench.py --config 5 --steps 50 > gpurun_out/fin3_t7.log 2>&1
timeout 1500 bash tools/profile_round.sh fin3 3 > gpurun_out/fin3_prof.log 2>&1
for f in gpurun_out/fin3_*.log; do echo $f; tail -1 $f | cut -c1-200; done
