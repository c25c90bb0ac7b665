mkdir -p gpurun_out
CPB_BENCH_TIMELINE=1 python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 > gpurun_out/tl.log 2> gpurun_out/tl.err; grep timeline gpurun_out/tl.err; tail -1 gpurun_out/tl.log | cut -c1-150
