mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shapes.py -m gpu -q > gpurun_out/pytest_ak.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ak.log; grep "^E \|FAILED" gpurun_out/pytest_ak.log | head -10
