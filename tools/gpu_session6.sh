set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 900 python tools/probe_sizes.py 296 4 1 2>&1 | tail -14
MGK_PANEL_CTAS_PER_SM=1 timeout 300 python tools/probe_sizes.py 296 0 2>&1 | tail -3
