python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in serial overlap; do
  if [ $v = serial ]; then X=--serial; else X=; fi
  python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 $X > gpurun_out/ab_$v.log 2>&1; echo "$v"; python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))"
done
