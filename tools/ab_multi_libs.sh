#!/bin/bash
# A/B/C... of in-tree library builds (paper_2509_19777_b200/libhplmm_<tag>.so) on op timings:
#   bash tools/ab_multi_libs.sh cfg3 "a pf2 pf4" SPMV
cfg=${1:-cfg3}; tags=${2:-"a b"}; shift 2; ops=${@:-SPMV}
for rep in 1 2; do
  for v in $tags; do
    echo "== $v $(HPLMM_LIB=$PWD/paper_2509_19777_b200/libhplmm_$v.so NOSOLVE=1 timeout 200 python tools/time_ops.py $cfg -- $ops 2>&1 | grep 'ms per' | tr '\n' ' ')"
  done
done
