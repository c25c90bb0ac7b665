#!/bin/bash
# build a library variant for same-box A/B: tools/build_variant.sh NAME "-DFOO=1 ..."
# -> ab/NAME.so (the in-tree library is rebuilt with default flags afterwards)
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
CPB_NVCC_EXTRA="$2" python -c "from paper_2407_18015_b200 import build; build.build(force=True)" > /tmp/cpb_variant.log 2>&1 || { tail -20 /tmp/cpb_variant.log; exit 1; }
cp paper_2407_18015_b200/libcritprob_b200.so ab/$1.so
grep -A2 "closed_fuse_uniform\|closed_hist_tab_kernelILi5\|closed_uniform_kernel\|closed_pp_kernelILb0" paper_2407_18015_b200/_build/ptxas.log | grep Used | head -4 | sed "s/^/$1: /"
