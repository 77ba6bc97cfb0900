#!/bin/bash
# A/B of k_sn_solve variants selected at run time by HPLMM_SN_FLAGS (see
# supernodal.cu): e.g. the L2 prefetch distance PD (flags 0x1000 | PD << 8).
#   bash tools/sn_flags_ab.sh cfg3 "4096 4352 4608 4864 5120 5632" MZETA MGRAIN
cfg=${1:-cfg3}; flagsets=${2:-"4096 4608"}; shift 2; ops=${@:-MZETA MGRAIN}
for rep in 1 2; do
  for f in $flagsets; do
    echo "== flags $f"
    HPLMM_SN_FLAGS=$f NOSOLVE=1 timeout 300 python tools/time_ops.py $cfg -- $ops 2>&1 | grep "ms per"
  done
done
