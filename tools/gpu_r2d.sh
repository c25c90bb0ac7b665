mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "semi or cases or engine" > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_d.log
timeout 300 python tools/bench_estimators.py 2>&1 | grep semi
VARIANTS="base nosweep" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
P="python bench.py --models histogram --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
$P > gpurun_out/prof_hist_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:closed_hist_tab -c 1 -o gpurun_out/prof_hist_r2d $P > gpurun_out/prof_hist_ncu.log 2>&1; tail -1 gpurun_out/prof_hist_ncu.log
