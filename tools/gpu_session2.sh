set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 600 python tools/probe_sizes.py 296 4 2>&1 | tail -10
MGK_NO_PANEL=1 timeout 300 python tools/probe_sizes.py 64 0 2>&1 | tail -4
