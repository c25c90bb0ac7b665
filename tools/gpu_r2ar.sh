mkdir -p gpurun_out
cp ab/ppnodiv.so paper_2407_18015_b200/libcritprob_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "epan or parity or slab or shapes" > gpurun_out/pytest_ar.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ar.log
VARIANTS="base ppnodiv" CMD="python bench.py --models epanechnikov --no-e2e --steps 5 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
