for v in "" t128; do
  if [ -n "$v" ]; then export MGK_LIB=paper_1910_06310_b200/libmgk_$v.so; fi
  echo "== variant ${v:-default}"
  timeout 600 python tools/probe_sizes.py 296 0 2>&1 | grep -E "pairs/s"
done
unset MGK_LIB
MGK_PANEL_SMEM_NM=16384 timeout 300 python tools/probe_sizes.py 296 0 2>&1 | grep -E "C5"
