# BASELINE config 3: histogram 2048 x 2048 x 40 members, bins 8 / 16 / 32 (closed form),
# one JSON line per bin count -> gpurun_out/config3_<tag>.jsonl
mkdir -p gpurun_out
out=gpurun_out/config3_${TAG:-x}.jsonl; : > $out
for b in 8 16 32; do
  python bench.py --height 2048 --width 2048 --members 40 --bins $b --models histogram --fit separate \
      --steps ${STEPS:-20} --warmup 3 --no-e2e ${EXTRA:-} > gpurun_out/config3_b$b.log 2>&1
  tail -1 gpurun_out/config3_b$b.log >> $out
  python -c "
import json,sys; d=json.loads(open('gpurun_out/config3_b$b.log').read().strip().splitlines()[-1])
print('bins $b', d['value'], 'Mvert/s', d['ms_per_step'], 'ms', json.dumps(d['roofline']['kernels']), 'parity', (d.get('parity') or {}).get('max_abs_err'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
