mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_aj.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_aj.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_aj.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_aj.log
timeout 600 python tools/run_reference_tests.py > gpurun_out/reftests_aj.log 2>&1; echo "reftests rc=$?"; tail -1 gpurun_out/reftests_aj.log | cut -c1-200
bash tools/gpu_r2t.sh
