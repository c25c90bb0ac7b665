# semianalytical A/B (tools/bench_estimators.py) over ab/<v>.so
cp paper_2407_18015_b200/libcritprob_b200.so /tmp/cpb_orig.so
for rep in 1 2; do for v in $VARIANTS; do
  cp ab/$v.so paper_2407_18015_b200/libcritprob_b200.so
  echo "$v $(python tools/bench_estimators.py 2>&1 | grep semi | head -1)"
done; done
cp /tmp/cpb_orig.so paper_2407_18015_b200/libcritprob_b200.so
