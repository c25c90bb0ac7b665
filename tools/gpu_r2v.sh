mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or fit_classify or uniform or slab or distributed or run_host" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v.log; grep "^E " gpurun_out/pytest_v.log | head -5
VARIANTS="base nohalo" CMD="python bench.py --models uniform --no-e2e --steps 10 --warmup 3" REPS=2 timeout 900 bash tools/ab.sh
P="python bench.py --models uniform --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:closed_fuse_edges -c 1 $P > gpurun_out/ncu_nohalo.log 2>&1; grep -E "duration|bytes" gpurun_out/ncu_nohalo.log | head
