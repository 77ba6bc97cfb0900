#!/bin/bash
# ncu launch list (duration + DRAM bytes) of one cfg solve, profiled region only.
# usage: tools/ncu_kernels.sh <cfg> <out.csv> [kernel-regex]
cfg=${1:-cfg3}; out=${2:-gpurun_out/ncu_kernels.csv}; re=${3:-.}
ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "regex:$re" --csv --log-file "$out" python tools/profile_solve.py "$cfg"
