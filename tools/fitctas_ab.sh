for v in 0 1 2; do python bench.py --no-e2e --no-cpu --steps 3 --warmup 2 --fit-ctas $v > gpurun_out/fc_v$v.log 2>&1; echo "fit_ctas=$v"; python -c "
import json; d=json.loads(open('gpurun_out/fc_v$v.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))"; done
python bench.py --no-e2e --no-cpu --steps 3 --warmup 2 --serial > gpurun_out/fc_serial.log 2>&1; echo serial; python -c "
import json; d=json.loads(open('gpurun_out/fc_serial.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))"
