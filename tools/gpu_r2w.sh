mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_w.log
bash tools/gpu_r2t.sh
