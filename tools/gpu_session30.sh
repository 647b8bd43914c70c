timeout 600 python tools/probe_sizes.py 0 4 1 2>&1 | grep -E "deg16|deg32"
MGK_GRID256=1 timeout 600 python tools/probe_sizes.py 0 4 1 2>&1 | grep -E "deg16|deg32"
