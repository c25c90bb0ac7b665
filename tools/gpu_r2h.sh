mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_h.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_h.log
VARIANTS="base ada" CMD="python bench.py --models epanechnikov --no-e2e --steps 5 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
grep -o '"max_abs_err": {[^}]*}' gpurun_out/ab_ada.log | head -2
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/cpb_keep.so
cp ab/boundscheck.so paper_2407_18015_b200/libcritprob_b200.so
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_boundscheck.log 2>&1; echo "boundscheck pytest rc=$?"; tail -3 gpurun_out/pytest_boundscheck.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_boundscheck.log 2>&1; echo "boundscheck smoke rc=$?"; tail -1 gpurun_out/smoke_boundscheck.log
grep -c "CPB_ASSERT failed" gpurun_out/pytest_boundscheck.log gpurun_out/smoke_boundscheck.log
cp /tmp/cpb_keep.so paper_2407_18015_b200/libcritprob_b200.so
