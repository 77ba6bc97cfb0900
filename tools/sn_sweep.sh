#!/bin/bash
# sweep of the supernodal solve on cfg3 (ncu launch durations + DRAM bytes)
# usage: tools/sn_sweep.sh "<chunk> <flags> <cfg>" ...   (cfg: 16 = 16 warps x 1 CTA, 8 = 8 x 2)
for cf in "$@"; do
  set -- $cf
  for op in MZETA MGRAIN; do
    HPLMM_SN_CHUNK=$1 HPLMM_SN_FLAGS=$2 HPLMM_SN_CFG=$3 timeout 300 ncu --profile-from-start off --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      --log-file gpurun_out/sn_${op}_$1_$2_$3.csv python tools/profile_apply.py cfg3 $op > gpurun_out/sn_${op}_$1_$2_$3.log 2>&1
  done
done
