python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-e2e --steps 2 --warmup 2 --models histogram --serial > gpurun_out/hist_ab.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/hist_ab.log').read().strip().splitlines()[-1]); print(json.dumps(d['roofline']['kernels']), d['parity'])"
