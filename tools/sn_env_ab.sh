#!/bin/bash
# A/B of k_sn_solve run-time variants given as environment settings, e.g.
#   bash tools/sn_env_ab.sh cfg3 "HPLMM_SN_CHUNK=4096|HPLMM_SN_CHUNK=2048 HPLMM_SN_FLAGS=4608" MZETA MGRAIN
cfg=${1:-cfg3}; sets=${2:-""}; shift 2; ops=${@:-MZETA MGRAIN}
IFS='|' read -ra V <<< "$sets"
for rep in 1 2; do
  for v in "${V[@]}"; do
    echo "== $v"
    env $v NOSOLVE=1 timeout 300 python tools/time_ops.py $cfg -- $ops 2>&1 | grep "ms per"
  done
done
