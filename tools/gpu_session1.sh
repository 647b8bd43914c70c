set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python tools/probe_sizes.py 64 1 2>&1 | tail -10
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_warp -c 1 -o gpurun_out/prof_warp python tools/prof_gram.py 800 1 > gpurun_out/ncu_warp.log 2>&1; tail -3 gpurun_out/ncu_warp.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-pairs 20000 2>&1 | tail -3
