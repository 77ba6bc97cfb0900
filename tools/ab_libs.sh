#!/bin/bash
# A/B timing of two in-tree builds of libhplmm (HPLMM_LIB selects the library):
#   cp paper_2509_19777_b200/libhplmm.so paper_2509_19777_b200/libhplmm_a.so   (variant a)
#   ... rebuild variant b ... cp ... libhplmm_b.so
#   bash tools/ab_libs.sh cfg3 MZETA MGRAIN
cfg=${1:-cfg3}; shift; ops=${@:-MZETA MGRAIN}
for v in a b a b; do
  echo "== $v"
  HPLMM_LIB=$PWD/paper_2509_19777_b200/libhplmm_$v.so NOSOLVE=1 timeout 200 \
    python tools/time_ops.py $cfg -- $ops 2>&1 | grep "ms per"
done
