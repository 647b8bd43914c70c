set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "pbr" 2>&1 | tail -5
timeout 900 python tools/probe_pbr.py c3 c4 2>&1 | tail -10
