for r in 0 4 8 16; do echo "rpc $r: $(MGK_PANEL_RPC=$r timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1)"; done
for c in 1 2 3; do echo "ctas/sm $c: $(MGK_PANEL_CTAS_PER_SM=$c timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1)"; done
