# Round-1 final measurement set (one GPU): bench lines for every config, the reference
# arm, and the ncu launch list / traffic / full captures of the headline bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin_smi.txt
timeout 900 python bench.py > gpurun_out/fin_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref.log 2>&1
timeout 600 python bench.py --config 0 --steps 20 > gpurun_out/fin_c1.log 2>&1
timeout 900 python bench.py --config 2 --steps 3 > gpurun_out/fin_c3.log 2>&1
timeout 900 python bench.py --config 3 --steps 2 --no-cpu-baseline > gpurun_out/fin_c4.log 2>&1
timeout 900 python bench.py --config 3 --dense-k 2 --steps 1 --no-cpu-baseline > gpurun_out/fin_c4_k2.log 2>&1
timeout 900 python bench.py --config 4 --virtual-ranks 2 --steps 3 > gpurun_out/fin_c5v2.log 2>&1
timeout 900 python bench.py --config 1 --dense-k 2 --steps 2 --no-cpu-baseline > gpurun_out/fin_c2_k2.log 2>&1
timeout 1500 bash tools/profile_round.sh fin 3 > gpurun_out/fin_prof.log 2>&1
for f in gpurun_out/fin_*.log; do echo $f; tail -1 $f | cut -c1-200; done
