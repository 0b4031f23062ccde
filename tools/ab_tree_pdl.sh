# A/B: the small trees' early prologue (programmatic launch) vs plain stream order; run on the GPU box as `bash tools/ab_tree_pdl.sh` after
#   python paper_2305_11645_b200/_build.py --variant nopdl -DRQMC_TREE_PDL=0
mkdir -p gpurun_out/s3g
for rep in 1 2; do for L in librqmc.so librqmc_nopdl.so; do
  for c in C1 C2; do echo "$c $L $(RQMC_LIB=$PWD/paper_2305_11645_b200/$L python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), "us", "e2e_us", round(d["config"]["N"]*d["config"]["tau"]/d["e2e"]["value"]*1e6,2))')" >> gpurun_out/s3g/ab.txt; done
  echo "C2x64 $L $(RQMC_LIB=$PWD/paper_2305_11645_b200/$L python bench.py --config C2 --replicas 64 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "ms")')" >> gpurun_out/s3g/ab.txt
done; done
python tools/timeline.py --config C2 --steps 2 > gpurun_out/s3g/timeline_C2.txt 2>&1
python tools/timeline.py --config C1 --steps 2 > gpurun_out/s3g/timeline_C1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_latency.py tests/test_gpu_fine_paths.py tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/s3g/t.log 2>&1; echo rc=$? >> gpurun_out/s3g/t.log
