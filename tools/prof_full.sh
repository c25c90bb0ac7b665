# round-end evidence at the bench's own config: launch list + ncu --set full of the hot kernels
F="python bench.py --no-e2e --no-cpu --steps 2 --warmup 3"
$F > gpurun_out/full_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-r1}.csv $F > gpurun_out/launch_ncu.log 2>&1
tail -1 gpurun_out/full_plain.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:"closed_hist_tab|closed_pp|closed_uniform|fit_tma" -s 8 -c 4 -o gpurun_out/prof_full_${TAG:-r1} $F > gpurun_out/prof_full_ncu.log 2>&1
tail -2 gpurun_out/prof_full_ncu.log
