mkdir -p gpurun_out
for m in epanechnikov histogram; do
  python bench.py --models $m --no-e2e --steps 10 --warmup 3 > gpurun_out/m.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m.log').read().strip().splitlines()[-1]); print('$m', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']), d['parity']['max_abs_err'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/m.log
done
