# gpurun session: GPU parity suite only (no -x: every failure listed).
#   gpurun --timeout 1500 -- 'bash tools/gpu_tests.sh [pytest args]'
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -q "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.log | tail -30
