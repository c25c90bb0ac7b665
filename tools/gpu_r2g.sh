# multi-model fit with 2 adjacent pixels per thread: parity with the pix2 build, then A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "multi or shapes or fit" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_g.log
VARIANTS="pix1 pix2" CMD="python bench.py --no-e2e --no-cpu --steps 5 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
