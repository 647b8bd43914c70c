mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
MGK_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
grep -E "k_pcg" gpurun_out/launches_c2.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150
run() { name=$1; shift; echo "== $name"; timeout 2400 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; tail -c 300 gpurun_out/bench_$name.json; tail -2 gpurun_out/bench_$name.err; }
run c2 --steps 3 --warmup 3
run c5 --config 5 --steps 1 --warmup 3
run c4 --config 4 --steps 1 --warmup 3
