set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/prof_gram.py 7165 2 2>&1 | tail -2
for v in "" s8p1 s4p0 s4p1; do
  if [ -n "$v" ]; then export MGK_LIB=paper_1910_06310_b200/libmgk_$v.so; fi
  echo "== variant ${v:-default}"
  timeout 600 python tools/probe_sizes.py 296 4 1 2>&1 | grep -E "pairs/s" | grep -v "deg4\|deg8"
done
