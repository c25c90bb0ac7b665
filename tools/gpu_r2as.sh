mkdir -p gpurun_out
VARIANTS="base hu2" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
