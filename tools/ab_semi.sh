# A/B of ab/base.so vs ab/new.so on the semianalytical estimator (tools/bench_estimators.py)
for v in base new base new; do
  cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
  python tools/bench_estimators.py 2>/dev/null | grep -i semi | sed "s/^/$v /"
done
cp ab/new.so paper_2407_18015_b200/libcritprob_b200.so
