mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/pytest_ai.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ai.log; grep "^E " gpurun_out/pytest_ai.log | head -3
