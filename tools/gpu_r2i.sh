# persistent-warp Epanechnikov stencil (+ L2 prefetch of the next segment): parity, then A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "epan or shapes or closed or golden or slab or count" > gpurun_out/pytest_i.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_i.log
VARIANTS="pp0 pp1 pp2" CMD="python bench.py --models epanechnikov --no-e2e --no-cpu --steps 5 --warmup 3" REPS=3 timeout 900 bash tools/ab.sh
