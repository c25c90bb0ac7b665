mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "epan or parity or slab or engine" > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_k.log
VARIANTS="base ada2 ada3" CMD="python bench.py --models epanechnikov --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_ada3.log | head -2
P="python bench.py --models epanechnikov --height 8192 --width 8192 --members 64 --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
cp ab/ada3.so paper_2407_18015_b200/libcritprob_b200.so
$P > gpurun_out/prof_pp_plain_ada3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:closed_pp -c 1 -o gpurun_out/prof_pp_ada3 $P > gpurun_out/prof_pp_ncu_ada3.log 2>&1; tail -1 gpurun_out/prof_pp_ncu_ada3.log
