# histogram sweep advancing only the tournament's arg-min list (ties -> zero-width pieces): parity, then A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "hist or shapes or closed or golden or slab" > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_l.log
VARIANTS="am0 am2" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
