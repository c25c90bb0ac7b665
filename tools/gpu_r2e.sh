mkdir -p gpurun_out
VARIANTS="old semi4 semi6 semi8" bash tools/ab_semi2.sh
VARIANTS="base h1" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
