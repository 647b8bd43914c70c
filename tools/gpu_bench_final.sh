mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() { name=$1; shift; echo "== $name"; timeout 2400 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 250 gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run c2 --steps 3 --warmup 3
run c3 --config 3 --steps 1 --warmup 3
run c5 --config 5 --steps 1 --warmup 3
