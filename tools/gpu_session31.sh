mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:k_pcg_panel --csv --log-file gpurun_out/traffic_c3.csv python tools/prof_pairs.py c3 296 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c3.csv gpurun_out/r01_ncu_summary_c3.json "k_pcg_panel" | tail -4
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_panel -c 1 -o gpurun_out/prof_panel512_c3 python tools/prof_pairs.py c3 296 > gpurun_out/ncu_panel512.log 2>&1; tail -1 gpurun_out/ncu_panel512.log
timeout 2400 python bench.py --config 4se --steps 1 --warmup 3 > gpurun_out/bench_c4se.json 2> gpurun_out/bench_c4se.err; tail -c 300 gpurun_out/bench_c4se.json; tail -3 gpurun_out/bench_c4se.err
