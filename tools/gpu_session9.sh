mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/prof_gram.py 7165 2 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
grep -E "k_pcg" gpurun_out/launches_c2.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_warp -c 2 -o gpurun_out/prof_warp2 python tools/prof_gram.py 800 1 > gpurun_out/ncu_warp2.log 2>&1; tail -2 gpurun_out/ncu_warp2.log
