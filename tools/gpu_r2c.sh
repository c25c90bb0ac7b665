mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "semi or cases or acceptance or engine" > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c.log
timeout 600 python tools/run_reference_tests.py > gpurun_out/reftests_c.log 2>&1; echo "reftests rc=$?"; tail -1 gpurun_out/reftests_c.log | cut -c1-400
timeout 300 python tools/bench_estimators.py > gpurun_out/est_c.log 2>&1; cat gpurun_out/est_c.log
python tools/small_field_timing.py
P="python bench.py --models histogram --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
$P > gpurun_out/prof_hist_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:closed_hist_tab -c 1 -o gpurun_out/prof_hist_r2c $P > gpurun_out/prof_hist_ncu.log 2>&1; tail -2 gpurun_out/prof_hist_ncu.log
