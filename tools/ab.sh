# A/B of two library builds on the same box: ab/base.so vs ab/new.so, each
# timed twice (alternating) with the bench command in $CMD (default: all models)
CMD=${CMD:-"python bench.py --no-e2e --no-cpu --steps 5 --warmup 3"}
for v in base new base new; do
  cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
  $CMD > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernels']))"
done
cp ab/new.so paper_2407_18015_b200/libcritprob_b200.so
