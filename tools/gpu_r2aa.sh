mkdir -p gpurun_out
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/cpb_orig.so
run() { python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 "$@" > gpurun_out/m.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m.log').read().strip().splitlines()[-1]); print('$V $*', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/m.log; }
for V in base h96; do
  cp ab/$V.so paper_2407_18015_b200/libcritprob_b200.so
  run
  run --fit fused-stencil --models uniform,histogram,epanechnikov
  run --fit fused-stencil
done
cp /tmp/cpb_orig.so paper_2407_18015_b200/libcritprob_b200.so
