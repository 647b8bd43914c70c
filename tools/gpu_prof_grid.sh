# ncu --set full of the grid solver on a small config-4 bucket (unlabeled, and SE-labeled).
mkdir -p gpurun_out
for v in "" se; do
  tag=grid${v}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_grid -c 1 \
    -o gpurun_out/prof_$tag -f python tools/prof_c4.py 8 1 4 $v > gpurun_out/prof_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_sass.csv 2>/dev/null
  ls -la gpurun_out/prof_$tag.*
done
