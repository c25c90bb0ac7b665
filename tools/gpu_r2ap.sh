mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py -m gpu -q > gpurun_out/pytest_ap.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ap.log; grep "^E " gpurun_out/pytest_ap.log | head -5
