mkdir -p gpurun_out
python bench.py --precision mixed --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_mixed_r2.log 2>&1; echo "mixed rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_mixed_r2.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['dtype'], json.dumps(d['roofline']['kernels']), d['parity']['max_abs_err'], d['parity']['tolerance'], d['clocks'])"
