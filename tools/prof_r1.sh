set -x
P="python bench.py --height 2048 --width 2048 --profile --no-e2e --no-cpu --steps 1 --warmup 0"
$P > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"closed_|fit_reg" -c 6 -o gpurun_out/prof_r1_small $P > gpurun_out/prof_ncu.log 2>&1
F="python bench.py --no-e2e --no-cpu --steps 2 --warmup 3"
$F > gpurun_out/full_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $F > gpurun_out/launch_ncu.log 2>&1
echo done
