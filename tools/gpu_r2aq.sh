mkdir -p gpurun_out
cp ab/unibl.so paper_2407_18015_b200/libcritprob_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "uniform or fused or parity or shapes" > gpurun_out/pytest_aq.log 2>&1; echo "pytest(unibl) rc=$?"; tail -1 gpurun_out/pytest_aq.log; grep "^E " gpurun_out/pytest_aq.log | head -3
VARIANTS="base unibl" CMD="python bench.py --no-e2e --no-cpu --steps 5 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
VARIANTS="base unibl" CMD="python bench.py --models uniform --no-e2e --no-cpu --steps 10 --warmup 3" REPS=2 timeout 1200 bash tools/ab.sh
