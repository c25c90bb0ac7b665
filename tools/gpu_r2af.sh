mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/pytest_af.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_af.log; grep "^E " gpurun_out/pytest_af.log | head -5
