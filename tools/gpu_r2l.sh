mkdir -p gpurun_out
VARIANTS="ada3 ada4" CMD="python bench.py --models epanechnikov --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_ada4.log | head -2
