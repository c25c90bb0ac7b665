mkdir -p gpurun_out
P="python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
cp ab/l2p2n.so paper_2407_18015_b200/libcritprob_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:fit_tma_multi -c 1 $P > gpurun_out/ncu_l2p2n.log 2>&1; grep -E "duration|bytes|issue" gpurun_out/ncu_l2p2n.log | head
cp ab/base.so paper_2407_18015_b200/libcritprob_b200.so
