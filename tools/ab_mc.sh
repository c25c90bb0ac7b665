# A/B of ab/base.so vs ab/new.so on the config-4 Monte Carlo (tools/bench_mc.py, splitmix64 lines)
for v in base new base new; do
  cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
  python tools/bench_mc.py 2>/dev/null | grep splitmix | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['model'], d['ms'], d['gdraws_per_s'], d['within_4se'])"
done
cp ab/new.so paper_2407_18015_b200/libcritprob_b200.so
