mkdir -p gpurun_out
VARIANTS="base fit64_5 fit64_6" CMD="python bench.py --no-e2e --no-cpu --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
