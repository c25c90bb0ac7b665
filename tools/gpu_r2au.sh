mkdir -p gpurun_out
for k in 5 10 20; do python bench.py --no-e2e --no-cpu --steps $k --warmup 3 > gpurun_out/k.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/k.log').read().strip().splitlines()[-1]); print('steps $k', d['value'], d['ms_per_step'])"; done
