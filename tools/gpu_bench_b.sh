mkdir -p gpurun_out
run() { name=$1; shift; echo "== $name"; timeout 2400 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 400 gpurun_out/bench_$name.json; tail -3 gpurun_out/bench_$name.err; }
run c5nw --config 5nw --steps 1 --warmup 3
run c3 --config 3 --steps 1 --warmup 3
run c4 --config 4 --steps 1 --warmup 3
run c4se --config 4se --count 8 --steps 1 --warmup 3
