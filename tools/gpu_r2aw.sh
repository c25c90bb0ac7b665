mkdir -p gpurun_out
for pri in -1 0; do
for order in uniform,epanechnikov,histogram histogram,epanechnikov,uniform epanechnikov,uniform,histogram; do
CPB_BENCH_FIT_PRIORITY=$pri CPB_BENCH_TIMELINE=1 python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 --models $order > gpurun_out/tl.log 2> gpurun_out/tl.err
echo "pri=$pri order=$order $(tail -1 gpurun_out/tl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; grep timeline gpurun_out/tl.err | sed -n 5,8p
done; done
