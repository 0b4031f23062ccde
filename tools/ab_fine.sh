#!/bin/bash
# A/B the fine kernel variants on the GPU box: parity subset + C5 phase times per library.
# usage: tools/ab_fine.sh lib1.so lib2.so ...   (default: librqmc.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for L in "${@:-paper_2305_11645_b200/librqmc.so}"; do
  echo "=== $L" >> gpurun_out/ab.log
  RQMC_LIB=$PWD/$L timeout 300 python -m pytest tests -m gpu -x -q -k "fine or C5 or parity" 2>&1 | tail -2 >> gpurun_out/ab.log
  RQMC_LIB=$PWD/$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'], d['qn'])" >> gpurun_out/ab.log 2>&1
done
