mkdir -p gpurun_out
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/cpb_keep.so
cp ab/boundscheck.so paper_2407_18015_b200/libcritprob_b200.so
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_boundscheck.log 2>&1; echo "boundscheck pytest rc=$?"; tail -2 gpurun_out/pytest_boundscheck.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_boundscheck.log 2>&1; echo "boundscheck smoke rc=$?"; tail -1 gpurun_out/smoke_boundscheck.log
echo "asserts fired: $(cat gpurun_out/pytest_boundscheck.log gpurun_out/smoke_boundscheck.log | grep -c 'CPB_ASSERT failed')"
cp /tmp/cpb_keep.so paper_2407_18015_b200/libcritprob_b200.so
