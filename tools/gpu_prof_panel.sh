# ncu --set full of the panel solver on a config-3 subset (shuffled proteins + device PBR), with the
# SASS source page for tools/ncu_by_line.py / tools/ncu_sass_top.py.
#   gpurun --timeout 1800 -- 'bash tools/gpu_prof_panel.sh [count] [tag]'
mkdir -p gpurun_out
N=${1:-150}
TAG=${2:-panel_c3}
timeout 300 python tools/prof_c3.py $N 2 2>&1 | tail -2
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_pcg_panel -c 1 \
  -o gpurun_out/prof_$TAG -f python tools/prof_c3.py $N 1 > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/prof_$TAG.*
