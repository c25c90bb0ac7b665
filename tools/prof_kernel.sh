# ncu --set full of selected kernels at 2048^2 after a clean plain run of the same command
# env: MODELS (default all), KREGEX (default closed_|fit_), TAG, COUNT (default 6)
P="python bench.py --height 2048 --width 2048 --profile --no-e2e --no-cpu --steps 1 --warmup 0 --models ${MODELS:-uniform,epanechnikov,histogram}"
$P > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-closed_|fit_}" -c ${COUNT:-6} -o gpurun_out/prof_${TAG:-x} $P > gpurun_out/prof_ncu.log 2>&1
tail -2 gpurun_out/prof_ncu.log
