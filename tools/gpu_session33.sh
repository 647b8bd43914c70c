timeout 900 python -m pytest tests -m gpu -x -q -k "pbr or reorder" 2>&1 | tail -2
bash tools/gpu_session32.sh
timeout 600 python tools/probe_pbr.py c3 2>&1 | tail -2
