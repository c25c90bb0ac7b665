mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "mixed or epan or parity" > gpurun_out/pytest_z.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_z.log
VARIANTS="base mxada" CMD="python bench.py --models epanechnikov --precision mixed --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_mxada.log | head -2
