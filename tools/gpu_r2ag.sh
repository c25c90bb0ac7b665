mkdir -p gpurun_out
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/keep.so
export CUDA_LAUNCH_BLOCKING=1
timeout 600 python -m pytest tests -m gpu -x -q -k "band_edges_and_degenerate" > gpurun_out/pytest_ag1.log 2>&1; echo "plain rc=$?"; grep "^E " gpurun_out/pytest_ag1.log | head -3
cp ab/boundscheck.so paper_2407_18015_b200/libcritprob_b200.so
timeout 600 python -m pytest tests -m gpu -x -q -s -k "band_edges_and_degenerate" > gpurun_out/pytest_ag2.log 2>&1; echo "boundscheck rc=$?"; grep -a "CPB_ASSERT\|^E " gpurun_out/pytest_ag2.log | head -5
cp /tmp/keep.so paper_2407_18015_b200/libcritprob_b200.so
