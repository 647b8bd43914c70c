mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 1500 gpurun_out/bench_c2.json; tail -4 gpurun_out/bench_c2.err
for r in 0 8 16; do echo "== rpc $r"; MGK_PANEL_RPC=$r timeout 300 python tools/probe_sizes.py 296 4 1 2>&1 | grep -E "C3:|C5|deg16|deg32"; done
timeout 1500 python bench.py --config 4 --count 8 --steps 1 --warmup 3 > gpurun_out/bench_c4_8.json 2> gpurun_out/bench_c4_8.err; tail -c 800 gpurun_out/bench_c4_8.json; tail -12 gpurun_out/bench_c4_8.err
