timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/probe_sizes.py 296 4 1 2>&1 | grep -E "pairs/s"
timeout 300 python tools/prof_c5.py 3000 2>&1 | tail -1
