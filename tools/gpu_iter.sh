# one GPU iteration: parity tests, a short full-size bench, ncu of the hot kernels at 2048^2
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -c 2500 gpurun_out/bench_full.log
if [ "${NCU:-0}" = "1" ]; then
P="python bench.py --height 2048 --width 2048 --profile --no-e2e --no-cpu --steps 1 --warmup 0"
$P > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"closed_|fit_" -c 6 -o gpurun_out/prof_${TAG:-x} $P > gpurun_out/prof_ncu.log 2>&1
tail -2 gpurun_out/prof_ncu.log
fi
