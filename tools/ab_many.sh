#!/bin/bash
# A/B of two in-tree builds (libhplmm_a.so / _b.so) on single and block applies
#   bash tools/ab_many.sh cfg3 4 MZETA MGRAIN
cfg=${1:-cfg3}; k=${2:-4}; shift 2; ops=${@:-MZETA MGRAIN}
for v in a b a b; do
  echo "== $v"
  HPLMM_LIB=$PWD/paper_2509_19777_b200/libhplmm_$v.so timeout 300 \
    python tools/time_many.py $cfg $k $ops 2>&1 | grep "block of"
done
