mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or parity or configs" > gpurun_out/pytest_ac.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ac.log
VARIANTS="base h96b" CMD="python bench.py --models histogram --no-e2e --steps 5 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_h96b.log | head -1
