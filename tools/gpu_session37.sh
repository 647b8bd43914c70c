timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1100 python tools/tiny_threshold.py 200 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 200 gpurun_out/bench_c2.json; tail -2 gpurun_out/bench_c2.err
