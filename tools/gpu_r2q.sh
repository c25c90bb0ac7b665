mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "epan or parity or slab" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_q.log
VARIANTS="base ada5 ada6" CMD="python bench.py --models epanechnikov --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_ada6.log | head -2
