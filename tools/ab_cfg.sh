#!/bin/bash
# A/B library variants on one config: tools/ab_cfg.sh CONFIG lib1.so lib2.so ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfg=$1; shift
for L in "$@"; do
  out=$(RQMC_LIB=$PWD/$L timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['phases_ms_per_step'].items()}, round(d['step_roofline']['frac'],4), d['qn'])" 2>&1)
  echo "$cfg $L $out" >> gpurun_out/ab_cfg.log
done
