#!/bin/bash
# per-launch device times of the coarse GEMMs (one C5 step) for each library variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in "$@"; do
  echo "=== $L" >> gpurun_out/ab_gemm.log
  RQMC_LIB=$PWD/$L timeout 300 python tools/prof_step.py --config C5 --steps 1 --warmup 1 > /dev/null 2>&1 || { echo "plain run failed" >> gpurun_out/ab_gemm.log; continue; }
  RQMC_LIB=$PWD/$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_level_gemm -s 7 -c 7 --csv python tools/prof_step.py --config C5 --steps 1 --warmup 1 2>/dev/null | grep gpu__time_duration | awk -F'","' '{print $(NF)}' | tr -d '"' | tr '\n' ' ' >> gpurun_out/ab_gemm.log
  echo >> gpurun_out/ab_gemm.log
done
