mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_f.log
timeout 600 python tools/run_reference_tests.py > gpurun_out/reftests_f.log 2>&1; echo "reftests rc=$?"; tail -1 gpurun_out/reftests_f.log | cut -c1-300
timeout 300 python tools/bench_estimators.py > gpurun_out/est_f.log 2>&1; cat gpurun_out/est_f.log
