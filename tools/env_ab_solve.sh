#!/bin/bash
# A/B of run-time variants (environment settings) on the full solve time:
#   bash tools/env_ab_solve.sh cfg3 "A=0|HPLMM_SN_FLAGS=1" [reps]
cfg=${1:-cfg3}; sets=${2:-"A=0"}; reps=${3:-2}
IFS='|' read -ra V <<< "$sets"
for rep in $(seq $reps); do
  for v in "${V[@]}"; do
    echo "== $v: $(env $v timeout 300 python tools/run_config.py $cfg 2>&1 | grep 'solve 1')"
  done
done
