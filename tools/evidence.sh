# Evidence pass (round 2): bench lines of every config, launch list and ncu summaries of C5,
# the C4 fine kernel, the C2 latency-regime kernels, kernel timelines of the small configs, the
# torchrun / gloo multi-rank dry runs and the simulated scaling.
# usage (on the GPU box): bash tools/evidence.sh r02a
P=${1:-r02}
set -x
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/${P}_bench_C5.json 2> gpurun_out/ev/bench_C5.err
for c in C1 C2 C3 C4 C5MC C3R C5U; do python bench.py --config $c > gpurun_out/ev/${P}_bench_$c.json 2> gpurun_out/ev/bench_$c.err; done
python bench.py --config C2 --replicas 64 > gpurun_out/ev/${P}_bench_C2_R64.json 2>/dev/null
python bench.py --config C3 --replicas 8 > gpurun_out/ev/${P}_bench_C3_R8.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev/${P}_bench_torchrun1.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/ev/${P}_bench_gloo2_dryrun.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/${P}_bench_reference.json 2>/dev/null
python tools/sim_scaling.py > gpurun_out/ev/${P}_sim_scaling_C5.json 2>/dev/null
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/${P}_launches_C5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
python tools/prof_step.py --config C5 > gpurun_out/ev/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_fine_tree|k_level_gemm|k_gen' -s 8 -c 9 -o gpurun_out/ev/${P}_C5_full python tools/prof_step.py --config C5 > gpurun_out/ev/ncu_full.log 2>&1
for c in C1 C2; do python tools/timeline.py --config $c --steps 2 > gpurun_out/ev/${P}_timeline_$c.txt 2>/dev/null; done
python tools/prof_step.py --config C2 > gpurun_out/ev/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_fine_tree|k_level_gemm_lat|k_gen' -s 12 -c 5 -o gpurun_out/ev/${P}_C2_full python tools/prof_step.py --config C2 --steps 1 --warmup 2 > gpurun_out/ev/ncu_c2.log 2>&1
python tools/prof_step.py --config C4 --xa > gpurun_out/ev/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_fine_tree' -c 1 -o gpurun_out/ev/${P}_C4_tree python tools/prof_step.py --config C4 --xa > gpurun_out/ev/ncu_c4.log 2>&1
ls -la gpurun_out/ev
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit)
python tools/ncu_summary.py launches gpurun_out/ev/${P}_launches_C5.csv "# ncu launch list, python bench.py --steps 2 --warmup 3 --no-cpu-baseline (C5), gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare SHARES" > gpurun_out/ev/${P}_launches_C5_summary.txt
python tools/ncu_summary.py full gpurun_out/ev/${P}_C5_full.ncu-rep "# ncu --set full --clock-control none --import-source on -k regex:'k_fine_tree|k_level_gemm|k_gen' -s 8 -c 9, tools/prof_step.py --config C5 (one step)" > gpurun_out/ev/${P}_ncu_C5_kernels.txt
python tools/ncu_summary.py full gpurun_out/ev/${P}_C2_full.ncu-rep "# ncu --set full, k_gen / k_level_gemm_lat / k_fine_tree of tools/prof_step.py --config C2 (one step)" > gpurun_out/ev/${P}_ncu_C2_kernels.txt
python tools/ncu_summary.py full gpurun_out/ev/${P}_C4_tree.ncu-rep "# ncu --set full, k_fine_tree of tools/prof_step.py --config C4 --xa (Y stored)" > gpurun_out/ev/${P}_ncu_C4_tree.txt
mkdir -p /tmp/ncurep && mv gpurun_out/ev/*.ncu-rep /tmp/ncurep/
du -sh gpurun_out
