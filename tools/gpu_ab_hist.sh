mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "semi or hist or cases or acceptance or engine" > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_b.log
timeout 600 python tools/run_reference_tests.py > gpurun_out/reftests_b.log 2>&1; echo "reftests rc=$?"; tail -3 gpurun_out/reftests_b.log
timeout 300 python tools/bench_estimators.py > gpurun_out/est_b.log 2>&1; cat gpurun_out/est_b.log
CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 10 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
