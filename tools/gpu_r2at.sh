mkdir -p gpurun_out
CPB_BENCH_HOSTTIME=1 python bench.py --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/ht.log 2> gpurun_out/ht.err; grep "host ms" gpurun_out/ht.err; tail -1 gpurun_out/ht.log | cut -c1-200
