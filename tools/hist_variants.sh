python -m pytest tests -m gpu -x -q -k "closed or hist" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in 0 1; do CPB_HIST_VARIANT=$v python bench.py --no-e2e --no-cpu --steps 2 --warmup 2 --models histogram > gpurun_out/hist_v$v.log 2>&1; echo "variant=$v"; python -c "
import json; d=json.loads(open('gpurun_out/hist_v$v.log').read().strip().splitlines()[-1]); print(json.dumps(d['roofline']['kernels']))"; done
