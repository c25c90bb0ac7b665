python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in 32 64 96; do CPB_FIT_STAGE_KB=$v python bench.py --no-e2e --no-cpu --steps 2 --warmup 2 > gpurun_out/fit_v$v.log 2>&1; echo "stage_kb=$v"; python -c "
import json; d=json.loads(open('gpurun_out/fit_v$v.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))"; done
