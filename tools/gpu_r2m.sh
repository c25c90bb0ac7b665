mkdir -p gpurun_out
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 "$@" > gpurun_out/m.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m.log').read().strip().splitlines()[-1]); print('$*', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))" || tail -3 gpurun_out/m.log; }
run
run --fit-ctas 1
run --fit-ctas 2
run --fit-ctas 3
run --models histogram,epanechnikov,uniform
run --models epanechnikov,histogram,uniform
run --models uniform,histogram,epanechnikov
run --serial
