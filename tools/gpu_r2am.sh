mkdir -p gpurun_out
VARIANTS="base minb5 minb6" CMD="python bench.py --models uniform --no-e2e --no-cpu --steps 10 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
