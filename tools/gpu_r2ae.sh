mkdir -p gpurun_out
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 "$@" > gpurun_out/m.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m.log').read().strip().splitlines()[-1]); print('$*', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/m.log; }
run
run --models histogram,epanechnikov,uniform
run --models histogram,uniform,epanechnikov
run --models histogram,epanechnikov,uniform --fit-ctas 2
run --models epanechnikov,histogram,uniform
