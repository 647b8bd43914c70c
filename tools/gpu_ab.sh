# A/B timing of libmgk variants (device solve time) on a config-2 Gram and a config-3 subset, after the
# GPU parity tests selected by $PYTEST_K (default: all; PYTEST_K=none skips them).
#   gpurun --timeout 1800 -- 'bash tools/gpu_ab.sh libmgk_old.so libmgk.so'
# AB_C2 / AB_C3 / AB_C4 (degree-8 bucket, unlabeled + SE) / AB_C5: graph counts (0 skips that workload); AB_PROF=1 adds ncu --set full of the panel solver
# on a 30-protein subset for every variant.
mkdir -p gpurun_out
if [ "${PYTEST_K:-}" != "none" ]; then
  K=${PYTEST_K:+-k $PYTEST_K}
  timeout 1200 python -m pytest tests -m gpu -q -x $K > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.log | tail -8
fi
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    [ "${AB_C2:-7165}" != 0 ] && MGK_LIB=paper_1910_06310_b200/$lib timeout 300 python tools/prof_gram.py ${AB_C2:-7165} 2 2>&1 | tail -1
    [ "${AB_C3:-150}" != 0 ] && MGK_LIB=paper_1910_06310_b200/$lib timeout 300 python tools/prof_c3.py ${AB_C3:-150} 2 2>&1 | tail -1
    [ "${AB_C4:-0}" != 0 ] && MGK_LIB=paper_1910_06310_b200/$lib timeout 300 python tools/prof_c4.py 8 1 ${AB_C4} 2>&1 | tail -1
    [ "${AB_C4:-0}" != 0 ] && MGK_LIB=paper_1910_06310_b200/$lib timeout 300 python tools/prof_c4.py 8 1 ${AB_C4} se 2>&1 | tail -1
    [ "${AB_C5:-0}" != 0 ] && MGK_LIB=paper_1910_06310_b200/$lib timeout 300 python tools/prof_c5.py ${AB_C5} 2>&1 | tail -1
  done
done
if [ -n "${AB_PROF:-}" ]; then
  for lib in "$@"; do
    tag=panel_c3_${lib%.so}
    MGK_LIB=paper_1910_06310_b200/$lib timeout 900 ncu --set full --import-source on --clock-control none \
      -k regex:k_pcg_panel -c 1 -o gpurun_out/prof_$tag -f python tools/prof_c3.py 30 1 > gpurun_out/prof_$tag.log 2>&1
    ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
    ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_sass.csv 2>/dev/null
    ls -la gpurun_out/prof_$tag.* | head -3
  done
fi
