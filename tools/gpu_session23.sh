mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 2400 python bench.py --config 5nw --steps 1 --warmup 3 > gpurun_out/bench_c5nw.json 2> gpurun_out/bench_c5nw.err; tail -c 300 gpurun_out/bench_c5nw.json; tail -3 gpurun_out/bench_c5nw.err
