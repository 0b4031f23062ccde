#!/bin/bash
# C2 (g = exp) batch/single timings per library variant and checkpoint override
cd "$(dirname "$0")/.."
for L in "$@"; do
  for ck in "" 2 6; do
    for r in 1 64; do
      out=$(RQMC_CKPT_W=$ck RQMC_LIB=$PWD/$L timeout 300 python bench.py --config C2 --replicas $r --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f'%d['ms_per_step'], '%.3g'%d['value'], {k:round(v,3) for k,v in d['phases_ms_per_step'].items()})" 2>&1)
      echo "$L ckpt=${ck:-auto} R=$r $out" >> gpurun_out/ab_c2.log
    done
  done
done
