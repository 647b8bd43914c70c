mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in 0 1; do echo "== tiny mode $m"; MGK_TINY_MODE=$m timeout 300 python tools/prof_gram.py 7165 2 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
grep -E "k_pcg" gpurun_out/launches_c2.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150
for m in 0 1; do MGK_TINY_MODE=$m timeout 1100 python tools/tiny_threshold.py 200 2>&1 | tail -3; done
