mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in paper_1910_06310_b200/libmgk.so paper_1910_06310_b200/libmgk_t1.so paper_1910_06310_b200/libmgk.so paper_1910_06310_b200/libmgk_t1.so; do
  echo $L; MGK_LIB=$PWD/$L timeout 300 python tools/prof_gram.py 7165 3 2>&1 | tail -1
done
for L in libmgk libmgk_t1; do
  MGK_LIB=$PWD/paper_1910_06310_b200/$L.so MGK_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pcg_tiny --csv --log-file gpurun_out/tiny_$L.csv python tools/prof_gram.py 7165 1 > /dev/null 2>&1
  echo $L; grep k_pcg_tiny gpurun_out/tiny_$L.csv | awk -F'","' '{print $(NF)}'
done
