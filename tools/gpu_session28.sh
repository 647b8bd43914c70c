for v in "" t512; do
  if [ -n "$v" ]; then export MGK_LIB=paper_1910_06310_b200/libmgk_$v.so; fi
  echo "== variant ${v:-default}"
  timeout 600 python tools/probe_sizes.py 296 0 2>&1 | grep -E "pairs/s"
  timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1
done
