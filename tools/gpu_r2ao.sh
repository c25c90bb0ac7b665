mkdir -p gpurun_out
export CPB_BENCH_BACKEND=gloo CPB_BENCH_SHARE_GPU=1
for args in "--gpus 2 --height 4096 --steps 2 --warmup 1" "--gpus 3 --height 2050 --steps 2 --warmup 1" "--gpus 2 --height 4096 --models uniform --steps 2 --warmup 1"; do
  timeout 900 python bench.py $args > gpurun_out/mr.log 2> gpurun_out/mr.err; rc=$?
  echo "== $args rc=$rc"; grep -c "process group" gpurun_out/mr.err
  python -c "
import json; d=json.loads(open('gpurun_out/mr.log').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels'])[:200], 'e2e', (d.get('e2e') or {}).get('value'), 'parity', (d.get('parity') or {}).get('max_abs_err'), (d.get('parity') or {}).get('ok'), 'cpu', d.get('cpu_baseline'))" || tail -5 gpurun_out/mr.err
done
