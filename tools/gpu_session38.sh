mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
MGK_SERIAL=1 timeout 600 ncu --metrics $M --clock-control none -k regex:k_pcg_warp --csv --log-file gpurun_out/traffic_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c2.csv gpurun_out/r01_ncu_summary_c2.json "k_pcg_warp<2, 0, 4>" | tail -3
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 2 --warmup 1 --cpu-pairs 2000 > gpurun_out/bench_under_ncu.log 2>&1
grep -c k_pcg gpurun_out/r01_bench_launches.csv
