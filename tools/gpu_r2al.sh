mkdir -p gpurun_out
P="python bench.py --models uniform --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
$P > gpurun_out/prof_fuse_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:closed_fuse -c 3 -o gpurun_out/prof_fuse_r2e $P > gpurun_out/prof_fuse_ncu.log 2>&1; tail -1 gpurun_out/prof_fuse_ncu.log
