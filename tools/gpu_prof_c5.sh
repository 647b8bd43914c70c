# Launch list (per-job kernel durations) of a config-5 subset Gram, then ncu --set full of its longest
# panel-solver launch, with the SASS source page.
#   gpurun --timeout 1800 -- 'bash tools/gpu_prof_c5.sh [count] [skip]'
mkdir -p gpurun_out
N=${1:-2000}
SKIP=${2:-0}
timeout 300 python tools/prof_c5.py $N 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic \
  --clock-control none -k regex:k_pcg --csv --log-file gpurun_out/launches_c5.csv python tools/prof_c5.py $N > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/launches_c5.csv")) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
idi = h.index("ID")
launch = {}
for r in rows[1:]:
    d = launch.setdefault(r[idi], {"k": r[ki][:60]})
    d[r[mi]] = r[vi]
for i, d in launch.items():
    print(i, d["k"], "ms", float(d.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e6,
          "grid", d.get("launch__grid_size"), "block", d.get("launch__block_size"),
          "dsmem", d.get("launch__shared_mem_per_block_dynamic"))
PY
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_pcg_panel -s $SKIP -c 1 \
  -o gpurun_out/prof_panel_c5 -f python tools/prof_c5.py $N > gpurun_out/prof_panel_c5.log 2>&1
ncu -i gpurun_out/prof_panel_c5.ncu-rep --page raw --csv > gpurun_out/prof_panel_c5_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_panel_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_panel_c5_sass.csv 2>/dev/null
ls -la gpurun_out/prof_panel_c5.*
