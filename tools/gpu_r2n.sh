mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or parity or engine or configs" > gpurun_out/pytest_n.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_n.log
VARIANTS="ada4 sort" CMD="python bench.py --models histogram --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_sort.log | head -2
