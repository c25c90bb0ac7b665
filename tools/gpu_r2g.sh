mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or smoke or parity" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_g.log
VARIANTS="base keys" CMD="python bench.py --models histogram --no-e2e --no-cpu --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
