mkdir -p gpurun_out
P="python bench.py --models epanechnikov --height 8192 --width 8192 --members 64 --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
for v in base ada; do
  cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
  $P > gpurun_out/prof_pp_plain_$v.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:closed_pp -c 1 -o gpurun_out/prof_pp_$v $P > gpurun_out/prof_pp_ncu_$v.log 2>&1; tail -1 gpurun_out/prof_pp_ncu_$v.log
done
cp ab/ada.so paper_2407_18015_b200/libcritprob_b200.so
