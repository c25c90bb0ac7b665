python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in 3 1; do CPB_PP=$v python bench.py --no-e2e --steps 2 --warmup 2 --models epanechnikov --serial > gpurun_out/epan_v$v.log 2>&1; echo "pp=$v"; python -c "
import json; d=json.loads(open('gpurun_out/epan_v$v.log').read().strip().splitlines()[-1]); print(json.dumps(d['roofline']['kernels']), d['parity'])"; done
