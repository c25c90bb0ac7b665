mkdir -p gpurun_out
VARIANTS="old new" CMD="python bench.py --models uniform --no-e2e --no-cpu --steps 10 --warmup 3" REPS=3 timeout 1200 bash tools/ab.sh
