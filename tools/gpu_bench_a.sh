mkdir -p gpurun_out
for c in 1 4 5; do
  echo "== config $c"
  timeout 1500 python bench.py --config $c --steps 1 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  tail -c 600 gpurun_out/bench_c$c.json; tail -3 gpurun_out/bench_c$c.err
done
