timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/prof_gram.py 7165 3 2>&1 | tail -1
MGK_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
grep -E "k_pcg" gpurun_out/launches_c2.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150
timeout 1100 python tools/tiny_threshold.py 200 2>&1 | tail -1
timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1
