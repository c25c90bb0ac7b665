# histogram list starts hoisted before the fast/exact branch: parity, then A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "hist or shapes or closed or golden or slab" > gpurun_out/pytest_h.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_h.log
VARIANTS="hoist0 hoist1" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
