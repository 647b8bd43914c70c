mkdir -p gpurun_out profiles
# 1. full ncu capture of the warp solvers on the whole config-2 Gram (roofline.traffic source)
MGK_SERIAL=1 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_pcg_warp -c 2 -o gpurun_out/prof_c2_full python tools/prof_gram.py 7165 1 > gpurun_out/ncu_c2_full.log 2>&1; tail -2 gpurun_out/ncu_c2_full.log
python tools/ncu_summary.py gpurun_out/prof_c2_full.ncu-rep profiles/r01_ncu_summary_c2.json "k_pcg_warp<2, 0, 4>" > gpurun_out/ncu_c2_summary.txt 2>&1; cat gpurun_out/ncu_c2_summary.txt | head -5; cp profiles/r01_ncu_summary_c2.json gpurun_out/
# 2. launch list of the bench command itself
MGK_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 2 --warmup 1 --cpu-pairs 2000 > gpurun_out/bench_under_ncu.log 2>&1; grep -c k_pcg gpurun_out/r01_bench_launches.csv
# 3. the bench line
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 700 gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
