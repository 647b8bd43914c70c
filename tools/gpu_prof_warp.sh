# Launch list (per-kernel durations) of a config-2 Gram, then ncu --set full of the narrow warp solver
# and the tiny solver on a config-2 subset, plus SASS-level source pages for tools/ncu_by_line.py.
#   gpurun --timeout 1800 -- 'bash tools/gpu_prof_warp.sh [count] [skipfull]'
mkdir -p gpurun_out
N=${1:-1500}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pcg --csv \
  --log-file gpurun_out/launches_c2.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
grep -o '"[^"]*k_pcg[^"]*","[^"]*","[^"]*","[^"]*","[^"]*","[^"]*","[^"]*","[^"]*","[^"]*","[^"]*"$' gpurun_out/launches_c2.csv | awk -F'","' '{print $1, $NF}' | cut -c1-60,200- | head
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/launches_c2.csv")) if len(r)>5 and "k_pcg" in r[4]]
for r in rows: print(r[4][:70], float(r[-1])/1e6, "ms")
PY
[ -n "$2" ] && exit 0
prof() {  # tag, kernel regex, launches to skip
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s $3 -c 1 \
    -o gpurun_out/prof_$1 -f python tools/prof_gram.py $N > gpurun_out/prof_$1.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$1_sass.csv 2>/dev/null
  ls -la gpurun_out/prof_$1.*
}
prof narrow k_pcg_warp 1
prof tiny k_pcg_tiny 0
