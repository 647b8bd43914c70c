# gpurun session: GPU parity suite + config-2 device Gram timing (3 reps) + serialized per-job timing.
#   gpurun --timeout 1800 -- 'bash tools/gpu_quick.sh [pytest -k expr]'
mkdir -p gpurun_out
if [ -n "$1" ]; then K="-k $1"; else K=""; fi
timeout 1300 python -m pytest tests -m gpu -q $K > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.log | tail -20
timeout 300 python tools/prof_gram.py 7165 3 2>&1 | tail -3
MGK_SERIAL=1 timeout 300 python tools/prof_gram.py 7165 2 2>&1 | tail -1
