# A/B of library builds on the same box: ab/<v>.so for v in $VARIANTS (default
# "base new"), alternating, $REPS rounds, with the bench command in $CMD
CMD=${CMD:-"python bench.py --no-e2e --no-cpu --steps 5 --warmup 3"}
VARIANTS=${VARIANTS:-"base new"}
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/cpb_orig.so
for rep in $(seq ${REPS:-2}); do
  for v in $VARIANTS; do
    cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
    $CMD > gpurun_out/ab_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']), d['clocks'].get('sm_mhz'))" || tail -3 gpurun_out/ab_$v.log
  done
done
cp /tmp/cpb_orig.so paper_2407_18015_b200/libcritprob_b200.so
